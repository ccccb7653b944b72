// Symbolic front end, part 5: the energy library used by the BASELINE configurations.
// Densities and registration helpers restate the reference's energies.hpp
// (/root/reference/proj/include/symel/energies.hpp) with identical expression construction,
// so the derived tapes are bit-identical to the reference's:
//   lame_from_young_poisson :23-30   tet_rule_* :38-47   inertia_energy :73-83
//   deformation_gradient_tet :86-91  deformation_gradient_tri :96-119
//   strain_energy_density :123-158   contact_barrier :165-167   tet_shape_gradients :357-388
//   add_inertia :418-430  add_solid_tet :435-461  add_fem_solid :465-519
//   add_membrane_tri :523-543  add_bending :594-609
// plus the point-triangle barrier that BASELINE config 5 needs (built through EnergyBuilder
// exactly like oracle/ref_driver.cpp does on the reference side).
#pragma once

#include <array>
#include <cmath>
#include <string>
#include <vector>

#include "symel/system.hpp"

namespace symel {

enum class Material { NH, StableNH, StVK, ARAP, FixedCorot };

struct MaterialParams {
  double mu = 0.0, lambda = 0.0;
  Material model = Material::StableNH;
};

inline MaterialParams lame_from_young_poisson(double young, double poisson, Material m = Material::StableNH) {
  return {young / (2.0 * (1.0 + poisson)), young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)), m};
}

struct QuadratureRule {
  std::vector<std::array<double, 4>> points;  // (w, xi, eta, zeta); weights sum to 1/6
};
inline QuadratureRule tet_rule_linear() { return {{{1.0 / 6.0, 0.25, 0.25, 0.25}}}; }
inline QuadratureRule tet_rule_quadratic() {
  const double a = 0.5854101966249685, b = 0.1381966011250105, w = 1.0 / 24.0;
  return {{{w, a, b, b}, {w, b, a, b}, {w, b, b, a}, {w, b, b, b}}};
}

inline Scalar inertia_energy(const Vector& x, const Vector& x0, const Vector& v0, const std::array<double, 3>& acc,
                             double dt, const Scalar& m) {
  if (dt == 0.0) throw Error("inertia_energy: dt must be nonzero");
  if (x.size() != 3 || x0.size() != 3 || v0.size() != 3) throw Error("inertia_energy: 3-component vectors required");
  Vector target(x.graph());
  for (std::size_t i = 0; i < 3; ++i) target.push_back(x0[i] + dt * v0[i] + dt * dt * acc[i]);
  return (m / (2.0 * dt * dt)) * (x - target).squared_norm();
}

// F = [x1-x0, x2-x0, x3-x0] [X1-X0, X2-X0, X3-X0]^-1
inline Matrix deformation_gradient_tet(const std::array<Vector, 4>& X, const std::array<Vector, 4>& x) {
  const Matrix Ds = Matrix::from_columns({x[1] - x[0], x[2] - x[0], x[3] - x[0]});
  const Matrix Dm = Matrix::from_columns({X[1] - X[0], X[2] - X[0], X[3] - X[0]});
  return Ds * Dm.inverse();
}

// 2x2 gradient of a triangle in its own orthonormal (thin-QR) frame times the rest inverse.
inline Matrix deformation_gradient_tri(const Matrix& Dm2inv, const std::array<Vector, 3>& x,
                                       double eps = kStableNormEps) {
  if (Dm2inv.rows() != 2 || Dm2inv.cols() != 2) throw Error("deformation_gradient_tri: 2x2 rest matrix required");
  ExprGraph& g = x[0].graph();
  const Vector e1 = x[1] - x[0], e2 = x[2] - x[0];
  const Scalar l1sq = e1.squared_norm();
  const Scalar l1 = stable_norm(e1, eps);
  const Scalar guard = l1sq - g.constant(eps * eps);
  const Scalar t = e1.dot(e2);
  const Scalar e2u = branch(guard, t / l1, g.constant(0.0));
  const Scalar proj = branch(guard, t / l1sq, g.constant(0.0));
  Vector perp(g);
  for (std::size_t i = 0; i < 3; ++i) perp.push_back(e2[i] - proj * e1[i]);
  const Scalar h = stable_norm(perp, eps);
  Matrix Ds2(g, 2, 2);
  Ds2.set(0, 0, l1);
  Ds2.set(0, 1, e2u);
  Ds2.set(1, 0, g.constant(0.0));
  Ds2.set(1, 1, h);
  return Ds2 * Dm2inv;
}

inline Scalar strain_energy_density(Material model, const Matrix& F, const Matrix* R, const Scalar& mu,
                                    const Scalar& lambda) {
  const int dim = F.rows();
  if (dim != F.cols() || (dim != 2 && dim != 3)) throw Error("strain_energy_density: F must be 2x2 or 3x3");
  ExprGraph& g = F.graph();
  const Scalar Ic = (F.transpose() * F).trace();
  const Scalar J = F.det();
  switch (model) {
    case Material::NH:
      return 0.5 * mu * (Ic - double(dim)) - mu * log(J) + 0.5 * lambda * pow(log(J), 2);
    case Material::StableNH: {
      if (dim != 3) throw Error("strain_energy_density: stable NH is 3x3 only");
      // Reparametrisation exactly as the reference (energies.hpp:136-138): lambda + 5/6 lambda.
      const Scalar mu_s = (4.0 / 3.0) * mu;
      const Scalar la_s = lambda + (5.0 / 6.0) * lambda;
      const Scalar alpha = 1.0 + mu_s / la_s - mu_s / (4.0 * la_s);
      return 0.5 * mu_s * (Ic - 3.0) + 0.5 * la_s * pow(J - alpha, 2) - 0.5 * mu_s * log(Ic + 1.0);
    }
    case Material::StVK: {
      const Matrix E = 0.5 * (F.transpose() * F - Matrix::identity(g, dim));
      return mu * E.frobenius_norm_sq() + 0.5 * lambda * pow(E.trace(), 2);
    }
    case Material::ARAP: {
      if (!R) throw Error("strain_energy_density: ARAP requires a rotation");
      const Scalar tr = (F.transpose() * (*R)).trace();
      return 0.5 * mu * (Ic - 2.0 * tr + double(dim)) + 0.5 * lambda * pow(J - 1.0, 2);
    }
    case Material::FixedCorot: {
      if (!R) throw Error("strain_energy_density: FixedCorot requires a rotation");
      const Matrix D = F - *R;
      return mu * D.frobenius_norm_sq() + 0.5 * lambda * pow(J - 1.0, 2);
    }
  }
  throw Error("strain_energy_density: unknown model");
}

// -k (d - dhat)^2 ln(d / dhat)
inline Scalar contact_barrier(const Scalar& d, const Scalar& d_hat, const Scalar& k) {
  return -(k * pow(d - d_hat, 2) * log(d / d_hat));
}

inline std::vector<std::array<Scalar, 3>> tet_shape_gradients(int nodes, const Scalar& xi, const Scalar& eta,
                                                              const Scalar& zeta) {
  ExprGraph& g = xi.graph();
  const Scalar one = g.constant(1.0);
  const std::array<Scalar, 4> lam = {one - xi - eta - zeta, xi, eta, zeta};
  static constexpr double gl[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  std::vector<std::array<Scalar, 3>> dN;
  if (nodes == 4) {
    for (int a = 0; a < 4; ++a) dN.push_back({g.constant(gl[a][0]), g.constant(gl[a][1]), g.constant(gl[a][2])});
    return dN;
  }
  if (nodes != 10) throw Error("tet_shape_gradients: 4 or 10 nodes");
  for (int a = 0; a < 4; ++a) {
    const Scalar c = 4.0 * lam[a] - 1.0;
    dN.push_back({c * gl[a][0], c * gl[a][1], c * gl[a][2]});
  }
  static constexpr int edges[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  for (const auto& e : edges) {
    std::array<Scalar, 3> r;
    for (int j = 0; j < 3; ++j) r[j] = 4.0 * (lam[e[0]] * gl[e[1]][j] + lam[e[1]] * gl[e[0]][j]);
    dN.push_back(r);
  }
  return dN;
}

inline EnergyHandle add_inertia(EnergySystem& sys, std::string name, ConnHandle verts, ArrayHandle x, ArrayHandle xp,
                                ArrayHandle v, ArrayHandle mass, double dt, const std::array<double, 3>& gravity) {
  if (dt == 0.0) throw Error("add_inertia: dt must be nonzero");
  return sys.add_energy(std::move(name), verts, [&](EnergyBuilder& b) {
    const Vector xs = b.bind(x, 0), x0 = b.bind(xp, 0), v0 = b.bind(v, 0);
    const Scalar m = b.bind_scalar(mass, 0);
    b.set(inertia_energy(xs, x0, v0, gravity, dt, m));
  });
}

inline EnergyHandle add_solid_tet(EnergySystem& sys, std::string name, ConnHandle tets, ArrayHandle x,
                                  ArrayHandle rest, Material model, const double& mu, const double& lambda) {
  if (model == Material::ARAP || model == Material::FixedCorot)
    throw Error("add_solid_tet: rotation-based models need a rotation array (not supported here)");
  return sys.add_energy(std::move(name), tets, [&](EnergyBuilder& b) {
    std::array<Vector, 4> xs, Xs;
    for (std::uint32_t a = 0; a < 4; ++a) xs[a] = b.bind(x, a);
    for (std::uint32_t a = 0; a < 4; ++a) Xs[a] = b.bind(rest, a);
    const Scalar smu = b.param(mu, "mu"), sla = b.param(lambda, "lambda");
    const Matrix F = deformation_gradient_tet(Xs, xs);
    const Matrix Dm = Matrix::from_columns({Xs[1] - Xs[0], Xs[2] - Xs[0], Xs[3] - Xs[0]});
    const Scalar Ve = Dm.det() / 6.0;
    b.set(Ve * strain_energy_density(model, F, nullptr, smu, sla));
  });
}

inline EnergyHandle add_fem_solid(EnergySystem& sys, std::string name, ConnHandle elems, ArrayHandle x,
                                  ArrayHandle rest, int nodes, const QuadratureRule& rule, Material model,
                                  const double& mu, const double& lambda) {
  if (nodes != 4 && nodes != 10) throw Error("add_fem_solid: 4 or 10 nodes per element");
  if (rule.points.empty()) throw Error("add_fem_solid: empty quadrature rule");
  double ws = 0.0;
  for (const auto& r : rule.points) {
    if (!(r[0] > 0.0)) throw Error("add_fem_solid: quadrature weights must be positive");
    ws += r[0];
  }
  if (std::abs(ws - 1.0 / 6.0) > 1e-12) throw Error("add_fem_solid: quadrature weights must sum to the reference volume");
  if (model == Material::ARAP || model == Material::FixedCorot)
    throw Error("add_fem_solid: rotation-based models need a rotation array (not supported here)");
  return sys.add_energy(std::move(name), elems, [&](EnergyBuilder& b) {
    std::vector<Vector> xs, Xs;
    for (int a = 0; a < nodes; ++a) xs.push_back(b.bind(x, std::uint32_t(a)));
    for (int a = 0; a < nodes; ++a) Xs.push_back(b.bind(rest, std::uint32_t(a)));
    const Scalar smu = b.param(mu, "mu"), sla = b.param(lambda, "lambda");
    std::vector<std::vector<double>> items;
    for (const auto& r : rule.points) items.push_back({r[0], r[1], r[2], r[3]});
    const Scalar total = b.sum_items(items, [&](const Vector& it) {
      const Scalar w = it[0];
      const auto dN = tet_shape_gradients(nodes, it[1], it[2], it[3]);
      ExprGraph& g = b.graph();
      Matrix J(g, 3, 3), jd(g, 3, 3);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          Scalar aJ = Xs[0][std::size_t(i)] * dN[0][std::size_t(j)];
          Scalar aj = xs[0][std::size_t(i)] * dN[0][std::size_t(j)];
          for (int a = 1; a < nodes; ++a) {
            aJ = aJ + Xs[std::size_t(a)][std::size_t(i)] * dN[std::size_t(a)][std::size_t(j)];
            aj = aj + xs[std::size_t(a)][std::size_t(i)] * dN[std::size_t(a)][std::size_t(j)];
          }
          J.set(i, j, aJ);
          jd.set(i, j, aj);
        }
      const Matrix F = jd * J.inverse();
      return strain_energy_density(model, F, nullptr, smu, sla) * w * J.det();
    });
    b.set(total);
  });
}

inline EnergyHandle add_membrane_tri(EnergySystem& sys, std::string name, ConnHandle tris, ArrayHandle x,
                                     ArrayHandle Dm2inv, ArrayHandle area, Material model, const double& mu,
                                     const double& lambda) {
  if (model == Material::ARAP || model == Material::FixedCorot)
    throw Error("add_membrane_tri: rotation-based models not supported for membranes");
  return sys.add_energy(std::move(name), tris, [&](EnergyBuilder& b) {
    std::array<Vector, 3> xs;
    for (std::uint32_t a = 0; a < 3; ++a) xs[a] = b.bind(x, a);
    const Vector dm = b.bind_element(Dm2inv);
    const Scalar Ae = b.bind_element_scalar(area);
    const Scalar smu = b.param(mu, "mu"), sla = b.param(lambda, "lambda");
    Matrix Dmi(b.graph(), 2, 2);
    Dmi.set(0, 0, dm[0]);
    Dmi.set(0, 1, dm[1]);
    Dmi.set(1, 0, dm[2]);
    Dmi.set(1, 1, dm[3]);
    b.set(Ae * strain_energy_density(model, deformation_gradient_tri(Dmi, xs), nullptr, smu, sla));
  });
}

// 0.5 k_b sum_ij Q_ij x_i x_j over a flap (x0, x1 shared edge; x2, x3 wings).
inline EnergyHandle add_bending(EnergySystem& sys, std::string name, ConnHandle flaps, ArrayHandle x, ArrayHandle Q,
                                const double& k_b) {
  return sys.add_energy(std::move(name), flaps, [&](EnergyBuilder& b) {
    Vector xe(b.graph());
    for (std::uint32_t a = 0; a < 4; ++a) {
      const Vector v = b.bind(x, a);
      for (std::size_t i = 0; i < 3; ++i) xe.push_back(v[i]);
    }
    const Vector q = b.bind_element(Q);
    const Scalar kb = b.param(k_b, "k_b");
    Scalar acc = b.constant(0.0);
    for (std::size_t i = 0; i < 12; ++i)
      for (std::size_t j = 0; j < 12; ++j) acc = acc + q[i * 12 + j] * xe[i] * xe[j];
    b.set(0.5 * kb * acc);
  });
}

// Point-triangle log barrier in offset form (BASELINE config 5):
// q_k = x[idx_k] + off_k, n = (q_b - q_a) x (q_c - q_a), d = n.(q_p - q_a) / |n|;
// active while d <= d_hat, line-search guard d > 0.
inline EnergyHandle add_contact_point_triangle(EnergySystem& sys, std::string name, ConnHandle pairs, ArrayHandle x,
                                               ArrayHandle offsets, const double& k_c, const double& d_hat) {
  return sys.add_energy(std::move(name), pairs, [&](EnergyBuilder& b) {
    std::array<Vector, 4> v;
    for (std::uint32_t k = 0; k < 4; ++k) v[k] = b.bind(x, k);
    const Vector o = b.bind_element(offsets);
    const Scalar kc = b.param(k_c, "k_c"), dh = b.param(d_hat, "d_hat");
    std::array<Vector, 4> q;
    for (std::size_t k = 0; k < 4; ++k) {
      Vector qk(b.graph());
      for (std::size_t i = 0; i < 3; ++i) qk.push_back(v[k][i] + o[3 * k + i]);
      q[k] = qk;
    }
    const Vector n = (q[2] - q[1]).cross(q[3] - q[1]);
    const Scalar d = n.dot(q[0] - q[1]) / n.norm();
    b.set(contact_barrier(d, dh, kc), d <= dh);
    b.set_guard(d);
  });
}

}  // namespace symel
