// TEST INFRASTRUCTURE ONLY -- proves the drop-in boundary in-process.
//
// Compiled against the UNMODIFIED reference headers (/root/reference/proj/include/symel, used
// in place, like ref_driver.cpp) plus include/symel_cuda_assembler.hpp, and linked to
// libsymel_cuda.so. It builds one reference EnergySystem from a case directory
// (ref_systems.hpp: the reference's own add_solid_tet / add_fem_solid / add_membrane_tri /
// add_bending / add_inertia / EnergyBuilder barrier), assembles it with the reference's CPU
// `symel::Assembler` (assembly.hpp:90-187) and with `symel::CudaAssembler` on the device, and
// compares them:
//   pattern (b, row_ptr, col_idx)  bit-exact
//   E, gradient, BCRS values       max|d| / max(1, |ref|_inf) <= tol  (acceptance_main.cpp:101-106)
// in the deterministic, atomic and ordered modes, then the reference's other entry points:
// energy_only, guard_min, active_count, pins (EnergySystem::pin), a topology change
// (set_elements on a subset), the check_finite error message, and -- with --spd -- the SPD
// projection (E and g unchanged; H symmetric). Prints one JSON line per check; exit code 0
// iff every check passed. Built by oracle/Makefile into oracle/_ref/ref_cuda_driver.
//
// usage: ref_cuda_driver CASE_DIR [--tol T] [--spd] [--threads N] [--exact ENERGY]
//   --exact: SYMEL_ENERGY_EXACT on that energy (the reference's rounding in every mode; for
//   ill-conditioned energies such as the point-triangle barrier at d ~ 1e-7 h)
#include <cmath>
#include <limits>
#include <thread>

#include "ref_systems.hpp"
#include "symel_cuda_assembler.hpp"

using namespace symel;

namespace {

int g_fail = 0;

double rel_err(const std::vector<double>& a, const std::vector<double>& ref) {
  if (a.size() != ref.size()) return std::numeric_limits<double>::infinity();
  double d = 0.0, m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double x = std::abs(a[i] - ref[i]);
    d = (x > d || std::isnan(x)) ? x : d;
    m = std::max(m, std::abs(ref[i]));
  }
  return d / std::max(1.0, m);
}

double rel_e(double a, double ref) { return std::abs(a - ref) / std::max(1.0, std::abs(ref)); }

// a JSON number (Python's json reads Infinity / NaN)
std::string jnum(double v) {
  if (std::isnan(v)) return "NaN";
  if (std::isinf(v)) return v > 0 ? "Infinity" : "-Infinity";
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

void report(const std::string& check, bool ok, const std::string& detail) {
  std::printf("{\"check\": \"%s\", \"ok\": %s, %s}\n", check.c_str(), ok ? "true" : "false", detail.c_str());
  std::fflush(stdout);
  if (!ok) ++g_fail;
}

struct Snapshot {
  double E = 0;
  std::vector<double> g;
  BcrsMatrix H;
};

Snapshot take_ref(Assembler& as) {
  Snapshot s;
  s.E = as.assemble();
  s.g = as.gradient();
  s.H = as.hessian();
  return s;
}

Snapshot take_dev(CudaAssembler& as) {
  Snapshot s;
  s.E = as.assemble();
  s.g = as.gradient();
  s.H = as.hessian();
  return s;
}

void compare(const std::string& check, const Snapshot& d, const Snapshot& r, double tol, bool values = true) {
  const bool pat = d.H.b == r.H.b && d.H.n_block_rows == r.H.n_block_rows && d.H.row_ptr == r.H.row_ptr &&
                   d.H.col_idx == r.H.col_idx;
  const double eE = rel_e(d.E, r.E), eg = rel_err(d.g, r.g), eH = values ? rel_err(d.H.values, r.H.values) : 0.0;
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "\"pattern_bit_exact\": %s, \"E\": %.17g, \"E_ref\": %.17g, \"err_E\": %.3e, \"err_g\": %.3e, "
                "\"err_H\": %.3e, \"blocks\": %zu, \"tol\": %.1e",
                pat ? "true" : "false", d.E, r.E, eE, eg, eH, d.H.n_blocks(), tol);
  report(check, pat && eE <= tol && eg <= tol && eH <= tol, buf);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_cuda_driver CASE_DIR [--tol T] [--spd] [--threads N]\n");
    return 2;
  }
  refcase::g_dir = argv[1];
  double tol = 1e-10;
  bool spd = false;
  std::string exact;
  int threads = static_cast<int>(std::thread::hardware_concurrency());
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--tol") tol = std::stod(argv[++i]);
    else if (a == "--spd") spd = true;
    else if (a == "--threads") threads = std::stoi(argv[++i]);
    else if (a == "--exact") exact = argv[++i];
    else { std::fprintf(stderr, "unknown option %s\n", a.c_str()); return 2; }
  }
  try {
    EnergySystem sys;
    const std::string kind = refcase::build_system(sys, false);
    KernelCache cache(refcase::g_dir + "/kcache", KernelBackend::interp);
    Assembler ref(sys, cache, std::max(1, threads), 8);
    CudaAssembler dev(sys, cache);
    std::vector<std::uint32_t> base_flags(sys.n_energies(), 0);
    for (std::size_t d = 0; d < sys.n_energies(); ++d)
      if (sys.energy_at(d).name == exact) dev.set_energy_flags(d, base_flags[d] = SYMEL_ENERGY_EXACT);
    const Snapshot r = take_ref(ref);

    // 1. the three device modes against the reference Assembler
    for (const auto& [name, mode] : {std::pair{"deterministic", CudaAssembleMode::deterministic},
                                     std::pair{"atomic", CudaAssembleMode::atomic},
                                     std::pair{"ordered", CudaAssembleMode::ordered}}) {
      dev.set_mode(mode);
      compare(std::string("assemble_") + name, take_dev(dev), r, mode == CudaAssembleMode::ordered ? 1e-13 : tol);
    }
    dev.set_mode(CudaAssembleMode::deterministic);
    take_dev(dev);

    // 2. energy_only / guard_min / active sets (assembly.hpp:130-173)
    {
      const double er = ref.energy_only(), ed = dev.energy_only();
      report("energy_only", rel_e(ed, er) <= tol,
             "\"E\": " + jnum(ed) + ", \"E_ref\": " + jnum(er) + ", \"err\": " + jnum(rel_e(ed, er)));
      const double gr = ref.guard_min(), gd = dev.guard_min();
      report("guard_min", gr == gd || rel_e(gd, gr) <= tol, "\"gmin\": " + jnum(gd) + ", \"gmin_ref\": " + jnum(gr));
      bool same = true;
      for (std::size_t d = 0; d < sys.n_energies(); ++d)
        same = same && ref.active_count(d) == dev.active_count(d) && ref.active(d) == dev.active(d);
      report("active_sets", same, "\"energies\": " + std::to_string(sys.n_energies()));
    }

    // 3. pins (EnergySystem::pin, apply_pins assembly.hpp:464-489)
    {
      const ArrayHandle x{0};
      sys.pin(x, 0);
      sys.pin(x, 1, 2);
      const Snapshot rp = take_ref(ref);
      compare("pins", take_dev(dev), rp, tol);
      sys.clear_pins();
    }

    // 4. SPD projection: E, g unchanged, H changes and stays exactly symmetric
    if (spd) {
      for (std::size_t d = 0; d < sys.n_energies(); ++d) dev.set_energy_flags(d, base_flags[d] | SYMEL_ENERGY_SPD);
      const Snapshot sd = take_dev(dev);
      compare("spd_energy_gradient", sd, r, tol, false);
      bool sym = true;
      const BcrsMatrix& H = sd.H;
      for (std::size_t row = 0; row < H.n_block_rows && sym; ++row)
        for (std::size_t k = H.row_ptr[row]; k < H.row_ptr[row + 1] && sym; ++k) {
          const std::size_t m = H.find_block(H.col_idx[k], row);
          for (int i = 0; i < H.b; ++i)
            for (int j = 0; j < H.b; ++j) sym = sym && H.block(k)[i * H.b + j] == H.block(m)[j * H.b + i];
        }
      report("spd_symmetric", sym, "\"blocks\": " + std::to_string(H.n_blocks()));
      for (std::size_t d = 0; d < sys.n_energies(); ++d) dev.set_energy_flags(d, base_flags[d]);
    }

    // 5. topology change: every other element of the first energy (stamp bump -> re-register)
    {
      const EnergyDef& def0 = sys.energy_at(0);
      const std::size_t ne = sys.n_elements(def0.conn);
      std::uint32_t arity = 0;
      bool per_element_arrays = false;  // bind_element arrays must keep one row per element
      for (const auto& s : def0.inputs) {
        if (s.kind == detail::InputKind::item_comp) arity = std::max(arity, s.tuple_slot + 1);
        per_element_arrays = per_element_arrays || s.kind == detail::InputKind::elem_comp;
      }
      const auto conn = refcase::read_bin<std::int64_t>("conn.i64");
      if (conn.size() == ne * arity && !per_element_arrays) {
        std::vector<std::int64_t> half;
        for (std::size_t e = 0; e < ne; e += 2) half.insert(half.end(), conn.begin() + e * arity, conn.begin() + (e + 1) * arity);
        sys.set_elements(def0.conn, half);
        compare("topology_change", take_dev(dev), take_ref(ref), tol);
        sys.set_elements(def0.conn, conn);
        compare("topology_restore", take_dev(dev), r, tol);
      }
    }

    // 6. check_finite: the same symel::Error message as the reference (assembly.hpp:426-438)
    {
      auto xs = sys.array_data(ArrayHandle{0});
      const std::vector<double> keep(xs.begin(), xs.end());
      xs[3 * 5 + 1] = std::numeric_limits<double>::quiet_NaN();
      std::string mr, md;
      try { ref.assemble(); } catch (const Error& e) { mr = e.what(); }
      try { dev.assemble(); } catch (const Error& e) { md = e.what(); }
      std::copy(keep.begin(), keep.end(), xs.begin());
      report("non_finite_message", !mr.empty() && mr == md, "\"ref\": \"" + mr + "\", \"dev\": \"" + md + "\"");
    }
  } catch (const std::exception& e) {
    std::printf("{\"check\": \"driver\", \"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return g_fail == 0 ? 0 : 1;
}
