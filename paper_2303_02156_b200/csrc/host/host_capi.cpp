// libsymel_host.so: C entry points of the C++ symbolic front end (symel/*.hpp) for tools that
// are not C++ (the Python tests and bench). The C++ API itself is header-only.
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "symel/materials.hpp"

namespace {

std::string g_err;

// Builds the energy named `kind` on a minimal system with the BASELINE configs' registration
// order (array ids as in paper_2303_02156_b200/systems.py) and returns its tapes.
std::map<std::string, std::vector<std::uint8_t>> build(const std::string& kind) {
  using namespace symel;
  static double mu = 1.0, lambda = 1.0, kb = 1.0, kc = 1.0, dhat = 1.0;
  EnergySystem sys;
  ArrayHandle x = sys.add_dof_array("x", 16, 3);
  ArrayHandle rest = sys.add_array("rest", 16, 3);
  std::string ename;
  if (kind == "tet4_elastic") {
    ConnHandle t = sys.add_connectivity("tets", 4);
    add_solid_tet(sys, "elastic", t, x, rest, Material::StableNH, mu, lambda);
  } else if (kind == "tet10_elastic") {
    ConnHandle t = sys.add_connectivity("tets", 10);
    add_fem_solid(sys, "elastic", t, x, rest, 10, tet_rule_quadratic(), Material::StableNH, mu, lambda);
  } else if (kind == "membrane") {
    ArrayHandle dm = sys.add_array("dm2inv", 1, 4), ar = sys.add_array("area", 1, 1);
    ConnHandle t = sys.add_connectivity("tris", 3);
    add_membrane_tri(sys, "membrane", t, x, dm, ar, Material::StVK, mu, lambda);
  } else if (kind == "bending") {
    ArrayHandle q = sys.add_array("Q", 1, 144);
    ConnHandle f = sys.add_connectivity("flaps", 4);
    add_bending(sys, "bending", f, x, q, kb);
  } else if (kind == "inertia") {
    ArrayHandle xp = sys.add_array("x_prev", 16, 3), v = sys.add_array("v", 16, 3), m = sys.add_array("mass", 16, 1);
    ConnHandle vc = sys.add_connectivity("verts", 1);
    add_inertia(sys, "inertia", vc, x, xp, v, m, 1.0 / 60.0, {0.0, 0.0, 0.0});
  } else if (kind == "contact") {
    ArrayHandle off = sys.add_array("pair_offset", 1, 12);
    ConnHandle pc = sys.add_connectivity("pairs", 4);
    add_contact_point_triangle(sys, "contact", pc, x, off, kc, dhat);
  } else {
    throw Error("unknown standard energy '" + kind + "'");
  }
  sys.compile_tapes();
  const EnergyDef& d = sys.energy_at(0);
  std::map<std::string, std::vector<std::uint8_t>> out;
  out["deriv"] = d.deriv->serialize();
  if (d.act) out["act"] = d.act->serialize();
  if (d.guard) out["guard"] = d.guard->serialize();
  return out;
}

}  // namespace

extern "C" {

// which: "deriv" | "act" | "guard". Two-call protocol: buf == NULL returns the size in *len.
int symel_host_standard_tape(const char* kind, const char* which, std::uint8_t* buf, std::uint64_t cap,
                             std::uint64_t* len) {
  try {
    const auto tapes = build(kind);
    auto it = tapes.find(which);
    if (it == tapes.end()) {
      g_err = std::string("energy '") + kind + "' has no '" + which + "' kernel";
      return 1;
    }
    *len = it->second.size();
    if (buf) {
      if (cap < it->second.size()) {
        g_err = "buffer too small";
        return 1;
      }
      std::memcpy(buf, it->second.data(), it->second.size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

const char* symel_host_last_error(void) { return g_err.c_str(); }

}  // extern "C"
