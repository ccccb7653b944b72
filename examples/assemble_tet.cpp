// The reference's user-facing flow, unchanged, on the B200 device path:
// declare an energy symbolically, bind arrays + connectivity, assemble.
//   build: see __graft_entry__.build() (examples/assemble_tet)
//   run:   examples/assemble_tet [n]   -> prints E, |g|_inf, BSR shape, CPU tape check of E
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "symel/assembler.hpp"
#include "symel/materials.hpp"

int main(int argc, char** argv) {
  using namespace symel;
  const int n = argc > 1 ? std::atoi(argv[1]) : 6;
  const int m = n + 1;
  EnergySystem sys;
  ArrayHandle x = sys.add_dof_array("x", std::size_t(m) * m * m, 3);
  ArrayHandle rest = sys.add_array("rest", std::size_t(m) * m * m, 3);
  std::mt19937_64 rng(0x5eed5eed);
  std::uniform_real_distribution<double> U(-0.3 / n, 0.3 / n);
  auto X = sys.array_data(rest);
  auto xs = sys.array_data(x);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      for (int k = 0; k < m; ++k) {
        const std::size_t id = (std::size_t(i) * m + j) * m + k;
        const double p[3] = {double(i) / n, double(j) / n, double(k) / n};
        for (int c = 0; c < 3; ++c) {
          X[3 * id + c] = p[c];
          xs[3 * id + c] = p[c] + U(rng);
        }
      }
  std::vector<std::int64_t> tets;  // Kuhn 6-tet split (cube_2.tet:29-40)
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        auto v = [&](int a, int b, int c) { return std::int64_t((std::size_t(i + a) * m + (j + b)) * m + (k + c)); };
        const std::int64_t T[6][4] = {{v(0, 0, 0), v(1, 0, 0), v(1, 1, 0), v(1, 1, 1)},
                                      {v(0, 0, 0), v(1, 0, 1), v(1, 0, 0), v(1, 1, 1)},
                                      {v(0, 0, 0), v(1, 1, 0), v(0, 1, 0), v(1, 1, 1)},
                                      {v(0, 0, 0), v(0, 1, 0), v(0, 1, 1), v(1, 1, 1)},
                                      {v(0, 0, 0), v(0, 0, 1), v(1, 0, 1), v(1, 1, 1)},
                                      {v(0, 0, 0), v(0, 1, 1), v(0, 0, 1), v(1, 1, 1)}};
        for (auto& t : T) tets.insert(tets.end(), t, t + 4);
      }
  ConnHandle tc = sys.add_connectivity("tets", 4);
  sys.set_elements(tc, tets);
  static double mu = 0, lambda = 0;
  const MaterialParams mp = lame_from_young_poisson(1e5, 0.4);
  mu = mp.mu;
  lambda = mp.lambda;
  add_solid_tet(sys, "elastic", tc, x, rest, Material::StableNH, mu, lambda);

  Assembler as(sys, 0, AssembleMode::deterministic);
  const double E = as.assemble();
  const auto& g = as.gradient();
  const BcrsMatrix& H = as.hessian();
  double gmax = 0;
  for (double v : g) gmax = std::max(gmax, std::abs(v));
  // CPU check of E through the front end's own tape interpreter (test aid)
  const EnergyDef& def = sys.energy_at(0);
  double Ecpu = 0;
  std::vector<double> in(def.n_inputs()), out(def.deriv->n_outputs);
  for (std::size_t e = 0; e < tets.size() / 4; ++e) {
    for (std::size_t s = 0; s < def.inputs.size(); ++s) {
      const InputSrc& src = def.inputs[s];
      if (src.kind == InputKind::param) in[s] = *src.host;
      else in[s] = sys.array_data(ArrayHandle{src.array})[std::size_t(tets[4 * e + src.tuple_slot]) * 3 + src.comp];
    }
    def.deriv->eval(in.data(), out.data());
    Ecpu += out[0];
  }
  std::printf("E %.17g E_cpu %.17g |g|inf %.6g blocks %zu rows %zu rel %.3e\n", E, Ecpu, gmax, H.n_blocks(),
              H.n_block_rows, std::abs(E - Ecpu) / std::max(1.0, std::abs(Ecpu)));
  return std::abs(E - Ecpu) <= 1e-10 * std::max(1.0, std::abs(Ecpu)) ? 0 : 1;
}
