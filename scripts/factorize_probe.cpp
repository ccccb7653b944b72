// Developer probe: factorise a tape, report op counts / live set, check numerics vs the
// original tape on random inputs. usage: factorize_probe TAPE n_dofs [emit kind mode]
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <iterator>
#include <random>
#include "../paper_2303_02156_b200/csrc/factorize.hpp"
#include "../paper_2303_02156_b200/csrc/codegen.hpp"
using namespace symel_cuda;
static void run(const TapeIR& t, const std::vector<double>& in, std::vector<double>& out) {
  std::vector<double> r(t.n_regs);
  for (unsigned k = 0; k < t.n_inputs; ++k) r[k] = in[k];
  for (size_t c = 0; c < t.consts.size(); ++c) r[t.n_inputs + c] = t.consts[c];
  for (auto& i : t.instrs) {
    double a = r[i.a], b = r[i.b], c = r[i.c], d = 0;
    switch (i.op) { case TOp::add: d = a + b; break; case TOp::sub: d = a - b; break; case TOp::mul: d = a * b; break;
      case TOp::div: d = a / b; break; case TOp::neg: d = -a; break; case TOp::pow_int: { d = 1; long long n = i.iarg; bool inv = n < 0; if (inv) n = -n; for (long long q = 0; q < n; ++q) d *= a; if (inv) d = 1 / d; } break;
      case TOp::sqrt: d = std::sqrt(a); break; case TOp::log: d = std::log(a); break; case TOp::sin: d = std::sin(a); break;
      case TOp::cos: d = std::cos(a); break; case TOp::branch: d = a >= 0 ? b : c; break; default: break; }
    r[i.dst] = d;
  }
  out.resize(t.out_regs.size());
  for (size_t k = 0; k < out.size(); ++k) out[k] = r[t.out_regs[k]];
}
int main(int argc, char** argv) {
  std::ifstream is(argv[1], std::ios::binary);
  std::vector<std::uint8_t> blob((std::istreambuf_iterator<char>(is)), {});
  TapeIR t = parse_tape(blob.data(), blob.size());
  unsigned n = atoi(argv[2]);
  std::vector<std::uint32_t> dofs(n); for (unsigned k = 0; k < n; ++k) dofs[k] = k;
  FactorizeInfo info;
  auto f = factorize_linear_frontier(t, dofs, &info);
  if (!f) { std::printf("no factorisation\n"); return 0; }
  std::printf("frontier m=%u n=%u ops %llu -> %llu  L nnz %u\n", info.frontier, info.n_dofs,
              (unsigned long long)info.ops_before, (unsigned long long)info.ops_after, info.l_nonzeros);
  // numerics: inputs = perturbed reference tet + params (tet4 layout: x 12, X 12, mu, lambda)
  std::mt19937_64 rng(1); std::uniform_real_distribution<double> U(-0.05, 0.05);
  double worst = 0;
  for (int trial = 0; trial < 50; ++trial) {
    std::vector<double> in(t.n_inputs, 0.0);
    const double X[12] = {0,0,0, 1,0,0, 0,1,0, 0,0,1};
    for (unsigned k = 0; k < t.n_inputs; ++k) in[k] = 0.5 + U(rng);
    if (t.n_inputs == 26) { for (int k = 0; k < 12; ++k) { in[12 + k] = X[k] * 0.1 + U(rng) * 0.01; in[k] = in[12 + k] * 1.1 + U(rng) * 0.01; } in[24] = 35714.28; in[25] = 142857.14; }
    std::vector<double> a, b; run(t, in, a); run(*f, in, b);
    double m = 0, d = 0; for (size_t k = 0; k < a.size(); ++k) { m = std::max(m, std::abs(a[k])); d = std::max(d, std::abs(a[k] - b[k])); }
    worst = std::max(worst, d / std::max(1.0, m));
  }
  std::printf("max rel err vs tape over 50 random elements: %.3e\n", worst);
  // reduced SPD form: H = W^T M W must reproduce the tape's Hessian
  FactorizeInfo si;
  if (auto fs = factorize_spd(t, dofs, &si)) {
    const unsigned m = si.frontier;
    double w2 = 0;
    for (int trial = 0; trial < 50; ++trial) {
      std::vector<double> in(t.n_inputs, 0.0);
      for (unsigned k = 0; k < t.n_inputs; ++k) in[k] = 0.5 + U(rng);
      if (t.n_inputs == 26) { const double X[12] = {0,0,0, 1,0,0, 0,1,0, 0,0,1}; for (int k = 0; k < 12; ++k) { in[12 + k] = X[k] * 0.1 + U(rng) * 0.01; in[k] = in[12 + k] * 1.1 + U(rng) * 0.01; } in[24] = 35714.28; in[25] = 142857.14; }
      std::vector<double> a, b; run(t, in, a); run(*fs, in, b);
      std::vector<double> M(m * m);
      size_t o = 1 + n;
      for (unsigned i = 0; i < m; ++i) for (unsigned j = i; j < m; ++j) M[i * m + j] = M[j * m + i] = b[o++];
      const double* W = &b[o];
      double mx = 0, d = 0;
      for (unsigned k = 0; k <= n; ++k) { mx = std::max(mx, std::abs(a[k])); d = std::max(d, std::abs(a[k] - b[k])); }
      for (unsigned r = 0; r < n; ++r) for (unsigned c = 0; c < n; ++c) {
        double h = 0; for (unsigned i = 0; i < m; ++i) for (unsigned j = 0; j < m; ++j) h += W[i * n + r] * M[i * m + j] * W[j * n + c];
        mx = std::max(mx, std::abs(a[1 + n + r * n + c])); d = std::max(d, std::abs(h - a[1 + n + r * n + c]));
      }
      w2 = std::max(w2, d / std::max(1.0, mx));
    }
    std::printf("spd form: ops %llu, max rel err of E, g, W^T M W vs tape: %.3e\n", (unsigned long long)si.ops_after, w2);
  }
  for (int sch : {1, 2}) {
    auto order = schedule_instrs(*f, sch);
    std::vector<long> last(f->n_regs, -1);
    unsigned base = f->first_op_reg();
    for (size_t p = 0; p < order.size(); ++p) { auto& in = f->instrs[order[p]]; unsigned o[3] = {in.a, in.b, in.c}; for (int q = 0; q < top_arity(in.op); ++q) last[o[q]] = std::max<long>(last[o[q]], p); }
    std::vector<int> ev(order.size() + 2, 0);
    for (size_t p = 0; p < order.size(); ++p) { long l = std::max<long>(last[base + order[p]], p); ev[p]++; ev[l + 1]--; }
    int cur = 0, mx = 0; for (size_t p = 0; p < order.size(); ++p) { cur += ev[p]; mx = std::max(mx, cur); }
    std::printf("schedule %d: max live %d\n", sch, mx);
  }
}
