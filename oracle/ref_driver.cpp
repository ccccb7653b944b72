// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// Driver that runs the UNMODIFIED reference implementation (header-only `symel`,
// /root/reference/proj/include/symel/*.hpp, included in place — nothing is copied)
// on a case directory written by paper_2303_02156_b200/configs.py, and dumps:
//   * the reference's own tapes (Tape::save, tape.hpp:225-245) for every kernel,
//   * E, gradient and the BCRS Hessian from Assembler::assemble()
//     (assembly.hpp:108-126), plus per-element kernel outputs for a sample,
//   * steady-state timings (the CPU baseline, `cpu_baseline.kind = "reference"`),
//   * with --solver: the reference's BcrsMatrix::matvec (assembly.hpp:43-57), block-Jacobi
//     inverse and pcg (optimizer.hpp:52-158) on the assembled Hessian (solver fixtures).
// Built by oracle/Makefile into oracle/_ref/ref_driver.
//
// usage: ref_driver CASE_DIR [--backend interp|source] [--threads T] [--lanes W]
//                   [--repeat K] [--no-dump] [--cache DIR] [--elem-sample N] [--solver]
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "symel/assembly.hpp"
#include "symel/energies.hpp"
#include "symel/mesh_io.hpp"
#include "symel/optimizer.hpp"

using namespace symel;

namespace {

std::string g_dir;

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

std::map<std::string, std::string> read_manifest() {
  std::ifstream is(g_dir + "/manifest.txt");
  if (!is) throw std::runtime_error("missing manifest.txt");
  std::map<std::string, std::string> m;
  std::string k, v;
  while (is >> k >> v) m[k] = v;
  return m;
}

double num(const std::map<std::string, std::string>& m, const char* k) {
  auto it = m.find(k);
  if (it == m.end()) throw std::runtime_error(std::string("manifest: missing ") + k);
  return std::stod(it->second);
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver CASE_DIR [options]\n");
    return 2;
  }
  g_dir = argv[1];
  std::string backend = "source", cache_dir = "/tmp/symel_ref_cache";
  int threads = static_cast<int>(std::thread::hardware_concurrency());
  int lanes = 8, repeat = 1;
  bool dump = true, solver = false;
  std::size_t elem_sample = 64;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() { return std::string(argv[++i]); };
    if (a == "--backend") backend = next();
    else if (a == "--threads") threads = std::stoi(next());
    else if (a == "--lanes") lanes = std::stoi(next());
    else if (a == "--repeat") repeat = std::stoi(next());
    else if (a == "--no-dump") dump = false;
    else if (a == "--cache") cache_dir = next();
    else if (a == "--elem-sample") elem_sample = std::stoul(next());
    else if (a == "--solver") solver = true;
    else { std::fprintf(stderr, "unknown option %s\n", a.c_str()); return 2; }
  }
  try {
    const auto man = read_manifest();
    const std::string kind = man.at("kind");
    EnergySystem sys;
    // parameters live here so EnergyBuilder::param pointers stay valid
    static double mu = 0, lambda = 0, kb = 0, kc = 0, dhat = 0;

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

    KernelCache cache(cache_dir, backend == "source" ? KernelBackend::source : KernelBackend::interp);
    Assembler as(sys, cache, threads, lanes);
    const double t0 = now_ms();
    double E = as.assemble();
    const double first_ms = now_ms() - t0;
    double best = 1e300, total = 0;
    as.reset_timings();
    for (int r = 0; r < repeat; ++r) {
      const double a = now_ms();
      E = as.assemble();
      const double dtm = now_ms() - a;
      best = std::min(best, dtm);
      total += dtm;
    }
    std::size_t n_elems = 0;
    for (std::size_t d = 0; d < sys.n_energies(); ++d) n_elems += as.active_count(d);
    std::printf("{\"kind\": \"%s\", \"E\": %.17g, \"n_elements\": %zu, \"threads\": %d, \"lanes\": %d, "
                "\"backend\": \"%s\", \"first_ms\": %.3f, \"best_ms\": %.3f, \"mean_ms\": %.3f, "
                "\"eval_ms\": %.3f, \"assemble_ms\": %.3f, \"repeat\": %d, \"n_blocks\": %zu}\n",
                kind.c_str(), E, n_elems, threads, lanes, backend.c_str(), first_ms, best,
                repeat ? total / repeat : 0.0, repeat ? as.timings().eval_ms / repeat : 0.0,
                repeat ? as.timings().assemble_ms / repeat : 0.0, repeat, as.hessian().n_blocks());
    if (!dump) return 0;

    write_bin("ref_E.f64", &E, 1);
    write_bin("ref_g.f64", as.gradient().data(), as.gradient().size());
    const BcrsMatrix& H = as.hessian();
    std::vector<std::int64_t> rp(H.row_ptr.begin(), H.row_ptr.end());
    std::vector<std::int64_t> ci(H.col_idx.begin(), H.col_idx.end());
    write_bin("ref_rowptr.i64", rp.data(), rp.size());
    write_bin("ref_colidx.i64", ci.data(), ci.size());
    write_bin("ref_vals.f64", H.values.data(), H.values.size());
    if (solver) {
      // probe vector, y = H probe; block-Jacobi inverses and PCG (rhs = -g) for three shifts
      const std::size_t n = H.n_rows();
      std::vector<double> probe(n), y(n);
      for (std::size_t i = 0; i < n; ++i) probe[i] = 1.0 + 0.5 * std::sin(0.37 * double(i)) - 0.25 * double(i % 7) / 7.0;
      H.matvec(probe, y, 1);
      write_bin("ref_probe.f64", probe.data(), n);
      write_bin("ref_matvec.f64", y.data(), n);
      double dmax = 0.0;
      for (std::size_t r = 0; r < H.n_block_rows; ++r) {
        const double* v = H.block(H.find_block(r, r));
        for (int i = 0; i < H.b; ++i) dmax = std::max(dmax, std::abs(v[i * H.b + i]));
      }
      const double taus[3] = {0.0, 0.1 * dmax, 10.0 * dmax};
      write_bin("ref_pcg_taus.f64", taus, 3);
      std::vector<double> rhs(n), x(n), inv;
      for (std::size_t i = 0; i < n; ++i) rhs[i] = -as.gradient()[i];
      std::ofstream ps(g_dir + "/ref_pcg.txt");
      for (int t = 0; t < 3; ++t) {
        detail::block_jacobi_inverse(H, taus[t], inv);
        write_bin("ref_bjinv_" + std::to_string(t) + ".f64", inv.data(), inv.size());
        for (const double tol : {1e-4, 1e-10}) {
          const PcgResult pr = pcg(H, taus[t], rhs, x, tol, static_cast<int>(n), 1);
          const std::string tag = std::to_string(t) + (tol > 1e-6 ? "_loose" : "_tight");
          write_bin("ref_pcg_x_" + tag + ".f64", x.data(), n);
          char buf[256];
          std::snprintf(buf, sizeof buf, "%s %d %d %d %.17g\n", tag.c_str(), pr.iters, int(pr.converged),
                        int(pr.neg_curvature), pr.rel_residual);
          ps << buf;
        }
      }
    }
    std::ofstream st(g_dir + "/ref_stats.txt");
    st << "b " << H.b << "\n";
    for (std::size_t d = 0; d < sys.n_energies(); ++d) {
      const EnergyDef& def = sys.energy_at(d);
      const Tape& t = def.deriv_kernel.tape();
      t.save(g_dir + "/ref_tape_" + def.name + ".sytp");
      if (def.has_activation()) def.act_kernel.tape().save(g_dir + "/ref_tape_" + def.name + "_act.sytp");
      if (def.has_guard()) def.guard_kernel.tape().save(g_dir + "/ref_tape_" + def.name + "_guard.sytp");
      const NodeId root[1] = {def.energy_root};
      std::vector<NodeId> wrt(def.dof_syms.begin(), def.dof_syms.end());
      const auto cs = compression_stats(*def.graph, std::span<const NodeId>(root, 1));
      st << "energy " << def.name << " n_inputs " << t.n_inputs << " n_outputs " << t.n_outputs
         << " n_instrs " << t.instrs.size() << " n_consts " << t.consts.size() << " n_regs "
         << t.n_regs << " digest " << t.digest.hex() << " energy_ops " << cs.plan_ops
         << " active " << as.active_count(d) << "\n";
      // per-element kernel outputs (with fixed-summation accumulation, assembly.hpp:400-413)
      const std::size_t ne = std::min<std::size_t>(elem_sample, sys.n_elements(def.conn));
      const std::size_t stride = t.n_outputs;
      std::vector<double> outs(ne * stride), in(def.n_inputs()), o(stride), acc(stride), scratch;
      for (std::size_t e = 0; e < ne; ++e) {
        if (def.is_sum) {
          bool first = true;
          for (const auto& row : def.sum_items) {
            sys.gather_element_inputs(def, e, row.data(), in.data());
            def.deriv_kernel.eval(in.data(), o.data(), scratch);
            if (first) { acc = o; first = false; }
            else for (std::size_t k = 0; k < stride; ++k) acc[k] += o[k];
          }
        } else {
          sys.gather_element_inputs(def, e, nullptr, in.data());
          def.deriv_kernel.eval(in.data(), acc.data(), scratch);
        }
        std::copy(acc.begin(), acc.end(), outs.begin() + static_cast<std::ptrdiff_t>(e * stride));
      }
      write_bin("ref_elem_" + def.name + ".f64", outs.data(), outs.size());
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver error: %s\n", e.what());
    return 1;
  }
  return 0;
}
