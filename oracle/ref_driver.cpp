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
//                   [--warmup W] [--repeat K] [--no-dump] [--cache DIR] [--elem-sample N] [--solver]
//   W untimed assemble() calls (>= 1; the first includes kernel build + pattern build and is
//   reported as first_ms), then K timed calls.
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

#include "ref_systems.hpp"
#include "symel/optimizer.hpp"

using namespace symel;
using refcase::g_dir;
using refcase::now_ms;
using refcase::write_bin;


int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver CASE_DIR [options]\n");
    return 2;
  }
  refcase::g_dir = argv[1];
  std::string backend = "source", cache_dir = "/tmp/symel_ref_cache";
  int threads = static_cast<int>(std::thread::hardware_concurrency());
  int lanes = 8, repeat = 1, warmup = 1;
  bool dump = true, solver = false;
  std::size_t elem_sample = 64;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() { return std::string(argv[++i]); };
    if (a == "--backend") backend = next();
    else if (a == "--threads") threads = std::stoi(next());
    else if (a == "--lanes") lanes = std::stoi(next());
    else if (a == "--repeat") repeat = std::stoi(next());
    else if (a == "--warmup") warmup = std::max(1, std::stoi(next()));
    else if (a == "--no-dump") dump = false;
    else if (a == "--cache") cache_dir = next();
    else if (a == "--elem-sample") elem_sample = std::stoul(next());
    else if (a == "--solver") solver = true;
    else { std::fprintf(stderr, "unknown option %s\n", a.c_str()); return 2; }
  }
  try {
    EnergySystem sys;
    const std::string kind = refcase::build_system(sys, dump);

    KernelCache cache(cache_dir, backend == "source" ? KernelBackend::source : KernelBackend::interp);
    Assembler as(sys, cache, threads, lanes);
    const double t0 = now_ms();
    double E = as.assemble();
    const double first_ms = now_ms() - t0;
    for (int w = 1; w < warmup; ++w) E = as.assemble();
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
    {  // the reference's text format (BcrsMatrix::dump, assembly.hpp:60-74)
      std::ofstream ds(g_dir + "/ref_dump.txt");
      H.dump(ds);
    }
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
