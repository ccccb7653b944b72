// Host-callable wrappers around the solver kernels in solver_kernels.cu:
// BCRS SpMV, block-Jacobi inverse, PCG iteration. All enqueue on `stream`; return cudaError_t.
#pragma once

namespace symel_cuda::dev {

// Device-resident PCG scalars (written by the last CTA of each reduction).
struct PcgScalars {
  double rz;    // r . z
  double rr;    // r . r
  double pq;    // p . (H + tau I) p
  double beta;  // rz_next / rz
  double rhs2;  // rhs . rhs
  int neg;      // non-positive curvature met
  int done;     // converged or negative curvature: later iterations are no-ops
  double rel;   // relative residual at the top of the last iteration run
  double tol;   // rel_tol
  int iters;    // completed iterations (PcgResult::iters)
  int converged;
};

// Work vectors of one context (n = n_rows * b doubles each) and reduction scratch.
struct SolverWork {
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
  double* inv = nullptr;       // block-Jacobi inverses, n_rows * b * b
  double* partials = nullptr;  // per-CTA partial sums, 2 * max_partials
  unsigned* ticket = nullptr;  // last-CTA counter (self-resetting)
  PcgScalars* sc = nullptr;
  int max_partials = 0;
  int vec_grid = 0;            // fixed grid of the vector kernels (deterministic sums)
  long long n = 0;             // allocated length
};

// y = A x (+ tau x); with dot_out, also dot(x, y) into *dot_out (device).
int bsr_spmv(int b, const int* row_ptr, const int* col_idx, const double* vals, const double* x, double* y,
             long long n_rows, double tau, SolverWork* w, double* dot_out, void* stream, PcgScalars* pcg = nullptr);
long long spmv_partials_needed(int b, long long n_rows);
// Inverse of each diagonal block + tau I, bit for bit as optimizer.hpp:52-90.
int block_jacobi_inverse(int b, const int* row_ptr, const int* col_idx, const double* vals, long long n_rows,
                         double tau, double* inv, void* stream);
// x = 0, r = rhs, z = M^-1 r, p = z, scalars rz, rr, rhs2 (w->inv must hold the inverses).
int pcg_init(int b, const double* rhs, SolverWork* w, long long n_rows, void* stream);
// One iteration, including the convergence check at its top (device side, so the host can
// enqueue many iterations between reads): q = (H + tau I) p, p.q, update x r z, rz rr beta, p.
int pcg_iteration(int b, const int* row_ptr, const int* col_idx, const double* vals, double tau, SolverWork* w,
                  long long n_rows, int it, void* stream);

}  // namespace symel_cuda::dev
