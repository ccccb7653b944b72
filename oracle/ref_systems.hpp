// TEST INFRASTRUCTURE ONLY -- shared by ref_driver.cpp (the reference's CPU Assembler) and
// ref_cuda_driver.cpp (the same reference EnergySystem through symel::CudaAssembler).
//
// Builds a reference `EnergySystem` (unmodified /root/reference/proj/include/symel headers)
// from a case directory written by paper_2303_02156_b200/configs.py (Case.write_case_dir):
// arrays and connectivity in the reference's registration order, energies through the
// reference's own helpers (add_solid_tet, add_fem_solid, add_membrane_tri, add_bending,
// add_inertia, energies.hpp:418-609) and the point-triangle barrier built with EnergyBuilder.
#pragma once

#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <span>
#include <string>
#include <vector>

#include "symel/assembly.hpp"
#include "symel/energies.hpp"
#include "symel/mesh_io.hpp"

namespace refcase {

using namespace symel;

inline std::string g_dir;

template <class T>
std::vector<T> read_bin(const std::string& name) {
  std::ifstream is(g_dir + "/" + name, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open " + name);
  is.seekg(0, std::ios::end);
  const std::size_t n = static_cast<std::size_t>(is.tellg()) / sizeof(T);
  is.seekg(0);
  std::vector<T> v(n);
  is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
  return v;
}

template <class T>
void write_bin(const std::string& name, const T* p, std::size_t n) {
  std::ofstream os(g_dir + "/" + name, std::ios::binary | std::ios::trunc);
  os.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}

inline std::map<std::string, std::string> read_manifest() {
  std::ifstream is(g_dir + "/manifest.txt");
  if (!is) throw std::runtime_error("missing manifest.txt");
  std::map<std::string, std::string> m;
  std::string k, v;
  while (is >> k >> v) m[k] = v;
  return m;
}

inline double num(const std::map<std::string, std::string>& m, const char* k) {
  auto it = m.find(k);
  if (it == m.end()) throw std::runtime_error(std::string("manifest: missing ") + k);
  return std::stod(it->second);
}

inline double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}


// parameters live here so EnergyBuilder::param pointers stay valid for the process
inline double mu = 0, lambda = 0, kb = 0, kc = 0, dhat = 0;

// Returns the case kind ("tet4", "tet10", "cloth", "contact").
inline std::string build_system(EnergySystem& sys, bool dump) {
  {
    const auto man = read_manifest();
    const std::string kind = man.at("kind");

    const std::vector<double> xs = read_bin<double>("x.f64");
    const std::vector<double> Xs = read_bin<double>("X.f64");
    const std::size_t nn = xs.size() / 3;
    ArrayHandle x = sys.add_dof_array("x", nn, 3);
    std::copy(xs.begin(), xs.end(), sys.array_data(x).begin());
    ArrayHandle rest = sys.add_array("rest", nn, 3);
    std::copy(Xs.begin(), Xs.end(), sys.array_data(rest).begin());
    mu = num(man, "mu");
    lambda = num(man, "lambda");

    if (kind == "tet4" || kind == "tet10" || kind == "contact") {
      const int npe = kind == "tet10" ? 10 : 4;
      ConnHandle tets = sys.add_connectivity("tets", static_cast<std::uint32_t>(npe));
      sys.set_elements(tets, read_bin<std::int64_t>("conn.i64"));
      if (kind == "tet10")
        add_fem_solid(sys, "elastic", tets, x, rest, 10, tet_rule_quadratic(),
                      Material::StableNH, mu, lambda);
      else
        add_solid_tet(sys, "elastic", tets, x, rest, Material::StableNH, mu, lambda);
    }
    if (kind == "contact") {
      const double dt = num(man, "dt");
      kc = num(man, "kappa");
      dhat = num(man, "dhat");
      ArrayHandle xprev = sys.add_array("x_prev", nn, 3);
      ArrayHandle vel = sys.add_array("v", nn, 3);
      ArrayHandle mass = sys.add_array("mass", nn, 1);
      const auto xp = read_bin<double>("x_prev.f64");
      const auto vv = read_bin<double>("v.f64");
      const auto mm = read_bin<double>("mass.f64");
      std::copy(xp.begin(), xp.end(), sys.array_data(xprev).begin());
      std::copy(vv.begin(), vv.end(), sys.array_data(vel).begin());
      std::copy(mm.begin(), mm.end(), sys.array_data(mass).begin());
      ConnHandle verts = sys.add_connectivity("verts", 1);
      std::vector<std::int64_t> vl(nn);
      for (std::size_t i = 0; i < nn; ++i) vl[i] = static_cast<std::int64_t>(i);
      sys.set_elements(verts, vl);
      add_inertia(sys, "inertia", verts, x, xprev, vel, mass, dt, {0.0, 0.0, 0.0});

      const auto pairs = read_bin<std::int64_t>("pairs.i64");
      const auto offs = read_bin<double>("offsets.f64");
      const std::size_t np = pairs.size() / 4;
      ConnHandle pc = sys.add_connectivity("pairs", 4);
      sys.set_elements(pc, pairs);
      ArrayHandle off = sys.add_array("pair_offset", np, 12);
      std::copy(offs.begin(), offs.end(), sys.array_data(off).begin());
      // Point-triangle log barrier, user-built through EnergyBuilder:
      // q_k = x[idx_k] + off_k, n = (q_b-q_a) x (q_c-q_a), d = n.(q_p-q_a)/|n|.
      sys.add_energy("contact", pc, [&](EnergyBuilder& b) {
        std::array<Vector, 4> v;
        for (int k = 0; k < 4; ++k) v[static_cast<std::size_t>(k)] = b.bind(x, static_cast<std::uint32_t>(k));
        const Vector o = b.bind_element(off);
        const Scalar skc = b.param(kc, "k_c");
        const Scalar sdh = b.param(dhat, "d_hat");
        std::array<Vector, 4> q;
        for (std::size_t k = 0; k < 4; ++k) {
          Vector qk(b.graph());
          for (std::size_t i = 0; i < 3; ++i) qk.push_back(v[k][i] + o[3 * k + i]);
          q[k] = qk;
        }
        const Vector nrm = (q[2] - q[1]).cross(q[3] - q[1]);
        const Scalar d = nrm.dot(q[0] - q[1]) / nrm.norm();
        b.set(contact_barrier(d, sdh, skc), d <= sdh);
        b.set_guard(d);
      });
    }
    if (kind == "cloth") {
      kb = num(man, "kb");
      const auto tris = read_bin<std::int64_t>("conn.i64");
      const std::size_t ne = tris.size() / 3;
      ConnHandle tc = sys.add_connectivity("tris", 3);
      sys.set_elements(tc, tris);
      ArrayHandle dm = sys.add_array("dm2inv", ne, 4);
      ArrayHandle area = sys.add_array("area", ne, 1);
      std::span<double> dmi = sys.array_data(dm);
      std::span<double> ar = sys.array_data(area);
      // Rest-frame rule restated from scene.hpp:783-805 (Scene is not buildable here).
      for (std::size_t e = 0; e < ne; ++e) {
        const std::int64_t* t = &tris[3 * e];
        double E1[3], E2[3];
        for (int c = 0; c < 3; ++c) {
          E1[c] = Xs[3 * std::size_t(t[1]) + std::size_t(c)] - Xs[3 * std::size_t(t[0]) + std::size_t(c)];
          E2[c] = Xs[3 * std::size_t(t[2]) + std::size_t(c)] - Xs[3 * std::size_t(t[0]) + std::size_t(c)];
        }
        const double L1 = std::sqrt(E1[0] * E1[0] + E1[1] * E1[1] + E1[2] * E1[2]);
        const double td = (E1[0] * E2[0] + E1[1] * E2[1] + E1[2] * E2[2]) / L1;
        double P[3];
        for (int c = 0; c < 3; ++c) P[c] = E2[c] - td / L1 * E1[c];
        const double h = std::sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
        dmi[4 * e + 0] = 1.0 / L1;
        dmi[4 * e + 1] = -td / (L1 * h);
        dmi[4 * e + 2] = 0.0;
        dmi[4 * e + 3] = 1.0 / h;
        ar[e] = 0.5 * L1 * h;
      }
      add_membrane_tri(sys, "membrane", tc, x, dm, area, Material::StVK, mu, lambda);
      const std::vector<std::int64_t> flaps = interior_edge_flaps(tris);
      const std::size_t nf = flaps.size() / 4;
      ConnHandle fc = sys.add_connectivity("flaps", 4);
      sys.set_elements(fc, flaps);
      ArrayHandle Q = sys.add_array("Q", nf, 144);
      std::span<double> Qd = sys.array_data(Q);
      for (std::size_t f = 0; f < nf; ++f) {
        std::array<std::array<double, 3>, 4> P;
        for (std::size_t k = 0; k < 4; ++k)
          for (std::size_t c = 0; c < 3; ++c) P[k][c] = Xs[3 * std::size_t(flaps[4 * f + k]) + c];
        const auto q = precompute_bending_Q(P[0], P[1], P[2], P[3]);
        std::copy(q.begin(), q.end(), Qd.begin() + static_cast<std::ptrdiff_t>(144 * f));
      }
      add_bending(sys, "bending", fc, x, Q, kb);
      if (dump) {
        write_bin("ref_flaps.i64", flaps.data(), flaps.size());
        write_bin("ref_dm2inv.f64", dmi.data(), dmi.size());
        write_bin("ref_area.f64", ar.data(), ar.size());
        if (nf <= 4096) write_bin("ref_Q.f64", Qd.data(), Qd.size());
      }
    }

    return kind;
  }
}

}  // namespace refcase
