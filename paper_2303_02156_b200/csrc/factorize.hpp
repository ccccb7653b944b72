// Tape-level optimisation for the fast kernels: linear-frontier factorisation of E, g, H.
//
// Many element energies reach their dofs only through an affine map y = L x + c (a linear
// tet's F = Ds Dm^-1: 9 values for 12 dofs; a quadratic tet's F at one quadrature point: 9
// values for 30 dofs; a membrane's edge vectors: 6 for 9). Writing E(x) = phi(y(x)),
//     g = L^T phi_y,     H = L^T phi_yy L,
// needs only the m(m+1)/2 second derivatives of phi (m = |y|) plus a sparse congruence,
// instead of the n(n+1)/2 forward-over-forward Hessian entries of the reference tape. The
// pass is generic: it re-imports the tape's energy closure into the symbolic engine, finds
// the affine frontier automatically (affine = add/sub/neg of affine nodes, affine times or
// divided by a dof-independent node), differentiates phi symbolically with the same rules
// as the front end (autodiff.hpp), and lowers the result back to a tape with the reference's
// output layout [E, g(n), H(n*n)]. Energies without a narrowing frontier are left untouched.
// The exact/ordered modes never use it (they execute the reference's own tape).
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "tape_io.hpp"

namespace symel_cuda {

struct FactorizeInfo {
  std::uint32_t frontier = 0;       // m = |y|
  std::uint32_t n_dofs = 0;
  std::uint64_t ops_before = 0, ops_after = 0;
  std::uint32_t l_nonzeros = 0;     // structurally nonzero entries of L = dy/dx
};

// Returns the factorised tape, or nothing when the energy has no narrowing affine frontier
// (m >= n) or the rewrite would not reduce the operation count.
std::optional<TapeIR> factorize_linear_frontier(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots,
                                                FactorizeInfo* info = nullptr);

// Reduced form for the SPD projection (K2). With G = L L^T = R R^T (Cholesky) and
// W = R^-1 L (orthonormal rows), H = W^T M W with M = R^T phi_yy R (m x m). Because W has
// orthonormal rows, the eigen-clamp of the n x n element Hessian equals W^T clamp(M) W -- an
// m x m eigenproblem instead of n x n, exactly. Output layout:
//   [E, g(n), M packed upper row-major (m(m+1)/2), W row-major (m x n)]
// (structurally zero W entries are constant-zero outputs).
std::optional<TapeIR> factorize_spd(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots,
                                    FactorizeInfo* info = nullptr);

}  // namespace symel_cuda
