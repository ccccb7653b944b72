// Consumer of the assembled BCRS Hessian on the device: y = A x, the
// block-Jacobi preconditioner and the PCG iteration of the reference's Newton solver
// (/root/reference/proj/include/symel/assembly.hpp:43-57, optimizer.hpp:52-158).
//
// The SpMV is HBM-bound (72 B of block values + 4 B of column index per 3x3 block, x gathers
// hit L2): G = 8 lanes per block row, each lane walks the row's blocks with stride G
// (consecutive lanes read consecutive blocks), then a fixed xor-shuffle tree sums the G
// partial rows.
// Dot products are deterministic: per-CTA partials in a fixed grid, summed in CTA order by the
// last CTA to finish (ticket counter), so results do not depend on scheduling. The
// block-Jacobi inverse reproduces the reference's adjugate formula bit for bit (no
// contraction: explicit _rn intrinsics).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "solver_ops.hpp"

namespace symel_cuda::dev {
namespace {

constexpr int kThreads = 256;

// Fixed-shape block reduction of one double; result valid in thread 0.
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) s += sh[i];
  __syncthreads();
  return s;
}

// Last-CTA finalisation: CTA partials (n_part of them, stride nv) are summed in CTA order by
// the last CTA; returns true in that CTA (all threads), with sums in out[0..nv).
__device__ bool finish_partials(double* partials, int nv, const double* mine, unsigned* ticket, double* out) {
  __shared__ bool last;
  __shared__ double sh[kThreads / 32];
  if (threadIdx.x == 0) {
    for (int v = 0; v < nv; ++v) partials[(size_t)blockIdx.x * nv + v] = mine[v];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  for (int v = 0; v < nv; ++v) {
    double s = 0.0;
    // fixed assignment: thread t sums partials t, t + T, ... in order; then the fixed tree
    for (unsigned c = threadIdx.x; c < gridDim.x; c += kThreads) s += ((volatile double*)partials)[(size_t)c * nv + v];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[v] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  __syncthreads();
  return true;
}

// y = A x (+ tau x); optionally the partial of dot(x, y) (PCG: p . q).
// With sc (PCG): first the convergence check of optimizer.hpp:133-137 on the current r.r --
// identical in every CTA (same inputs); CTA 0 records it -- and nothing more once done.
template <int B, int G>
__global__ void __launch_bounds__(kThreads) k_spmv(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                                                   const double* __restrict__ vals, const double* __restrict__ x,
                                                   double* __restrict__ y, long long n_rows, double tau,
                                                   double* partials, unsigned* ticket, double* dot_out,
                                                   PcgScalars* sc) {
  __shared__ double sh[kThreads / 32];
  if (sc) {
    if (sc->done) return;
    const double rel = sqrt(sc->rr) / sqrt(sc->rhs2);
    if (rel <= sc->tol) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->rel = rel;
        sc->converged = 1;
        sc->done = 1;
      }
      return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->rel = rel;
  }
  const long long row = (long long)blockIdx.x * (kThreads / G) + threadIdx.x / G;
  const int lane = threadIdx.x % G;
  double acc[B];
#pragma unroll
  for (int i = 0; i < B; ++i) acc[i] = 0.0;
  if (row < n_rows) {
    const int k0 = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
    for (int k = k0 + lane; k < k1; k += G) {
      const int c = __ldg(col_idx + k);
      const double* v = vals + (long long)k * B * B;
      double xc[B];
#pragma unroll
      for (int j = 0; j < B; ++j) xc[j] = __ldg(x + (long long)c * B + j);
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) acc[i] = fma(__ldg(v + i * B + j), xc[j], acc[i]);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < B; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  double d = 0.0;
  if (row < n_rows && lane < B) {
    double yi = acc[0];
#pragma unroll
    for (int i = 1; i < B; ++i) if (lane == i) yi = acc[i];
    const double xi = x[row * B + lane];
    if (tau != 0.0) yi += tau * xi;  // (H + tau I) p, optimizer.hpp:139-140
    y[row * B + lane] = yi;
    d = xi * yi;
  }
  if (dot_out) {  // one partial per CTA; k_sum_partials adds them in CTA order
    const double s = block_sum(d, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

// Fixed-order sum of n partials by one 1024-thread CTA (deterministic, no atomics): thread t
// keeps four interleaved accumulators over c = t + 1024 k (independent loads in flight), then
// a fixed tree.
constexpr int kSumThreads = 1024;
__global__ void __launch_bounds__(kSumThreads) k_sum_partials(const double* __restrict__ partials, int n,
                                                              double* out, const PcgScalars* sc) {
  __shared__ double sh[kSumThreads / 32];
  if (sc && sc->done) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int c = threadIdx.x;
  for (; c + 3 * kSumThreads < n; c += 4 * kSumThreads) {
    a0 += __ldg(partials + c);
    a1 += __ldg(partials + c + kSumThreads);
    a2 += __ldg(partials + c + 2 * kSumThreads);
    a3 += __ldg(partials + c + 3 * kSumThreads);
  }
  for (; c < n; c += kSumThreads) a0 += __ldg(partials + c);
  double v = (a0 + a1) + (a2 + a3);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = sh[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *out = v;
  }
}

template <int B>
__global__ void k_bj_inverse(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                             const double* __restrict__ vals, long long n_rows, double tau, double* __restrict__ inv) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double* out = inv + r * B * B;
#pragma unroll
  for (int q = 0; q < B * B; ++q) out[q] = 0.0;
  int lo = row_ptr[r], hi = row_ptr[r + 1];
  const int end = hi;
  while (lo < hi) {  // find_block (assembly.hpp:33-39)
    const int m = (lo + hi) >> 1;
    if (col_idx[m] < r) lo = m + 1; else hi = m;
  }
  if (lo >= end || col_idx[lo] != r) {
#pragma unroll
    for (int i = 0; i < B; ++i) out[i * B + i] = 1.0;
    return;
  }
  const double* v = vals + (long long)lo * B * B;
  if (B == 1) {
    const double d = __dadd_rn(v[0], tau);
    out[0] = (isfinite(d) && d != 0.0) ? 1.0 / d : 1.0;
    return;
  }
  double m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) m[i * 3 + j] = __dadd_rn(v[i * 3 + j], i == j ? tau : 0.0);
  // optimizer.hpp:74-87 without contraction (the reference builds with -ffp-contract=off)
  auto mm = [](double a, double b, double c, double d) { return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d)); };
  const double det = __dadd_rn(__dsub_rn(__dmul_rn(m[0], mm(m[4], m[8], m[5], m[7])),
                                         __dmul_rn(m[1], mm(m[3], m[8], m[5], m[6]))),
                               __dmul_rn(m[2], mm(m[3], m[7], m[4], m[6])));
  if (!isfinite(det) || fabs(det) < 1e-300) {
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i * 3 + i] = 1.0;
    return;
  }
  const double id = 1.0 / det;
  out[0] = __dmul_rn(mm(m[4], m[8], m[5], m[7]), id);
  out[1] = __dmul_rn(mm(m[2], m[7], m[1], m[8]), id);
  out[2] = __dmul_rn(mm(m[1], m[5], m[2], m[4]), id);
  out[3] = __dmul_rn(mm(m[5], m[6], m[3], m[8]), id);
  out[4] = __dmul_rn(mm(m[0], m[8], m[2], m[6]), id);
  out[5] = __dmul_rn(mm(m[2], m[3], m[0], m[5]), id);
  out[6] = __dmul_rn(mm(m[3], m[7], m[4], m[6]), id);
  out[7] = __dmul_rn(mm(m[1], m[6], m[0], m[7]), id);
  out[8] = __dmul_rn(mm(m[0], m[4], m[1], m[3]), id);
}

// z = M^-1 r for one block row (detail::block_apply, optimizer.hpp:92-103)
template <int B>
__device__ __forceinline__ void bj_apply_row(const double* __restrict__ inv, const double* r, double* z, long long row) {
  const double* m = inv + row * B * B;
  double rv[B];
#pragma unroll
  for (int j = 0; j < B; ++j) rv[j] = r[row * B + j];
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) acc = fma(m[i * B + j], rv[j], acc);
    z[row * B + i] = acc;
  }
}

// PCG start (optimizer.hpp:127-133): x = 0, r = rhs, z = M^-1 r, p = z; sums r.z and r.r.
template <int B>
__global__ void __launch_bounds__(kThreads) k_pcg_init(const double* __restrict__ rhs, const double* __restrict__ inv,
                                                       double* x, double* r, double* z, double* p, long long n_rows,
                                                       double* partials, unsigned* ticket, PcgScalars* sc) {
  __shared__ double sh[kThreads / 32];
  double rz = 0.0, rr = 0.0;
  for (long long row = (long long)blockIdx.x * kThreads + threadIdx.x; row < n_rows; row += (long long)gridDim.x * kThreads) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      r[row * B + i] = rhs[row * B + i];
      x[row * B + i] = 0.0;
    }
    bj_apply_row<B>(inv, r, z, row);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      p[row * B + i] = z[row * B + i];
      rz = fma(r[row * B + i], z[row * B + i], rz);
      rr = fma(r[row * B + i], r[row * B + i], rr);
    }
  }
  double s[2] = {block_sum(rz, sh), block_sum(rr, sh)};
  double out[2];
  if (finish_partials(partials, 2, s, ticket, out) && threadIdx.x == 0) {
    sc->rz = out[0];
    sc->rr = out[1];
    sc->rhs2 = out[1];
    sc->neg = 0;
    sc->done = out[1] == 0.0;  // zero rhs: converged with x = 0 (optimizer.hpp:124-128)
    sc->converged = sc->done;
    sc->iters = 0;
    sc->rel = 0.0;
  }
}

// One PCG update after q = (H + tau I) p and p.q (optimizer.hpp:141-156). Non-positive
// curvature: flag it, and at iteration 0 return the preconditioned rhs (x = z).
template <int B>
__global__ void __launch_bounds__(kThreads) k_pcg_update(const double* __restrict__ inv, double* x, double* r, double* z,
                                                         const double* __restrict__ p, const double* __restrict__ q,
                                                         long long n_rows, int it, double* partials, unsigned* ticket,
                                                         PcgScalars* sc) {
  __shared__ double sh[kThreads / 32];
  if (sc->done) return;
  const double pq = sc->pq, rz_old = sc->rz;
  const long long stride = (long long)gridDim.x * kThreads;
  if (!(pq > 0.0)) {
    if (it == 0)
      for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n_rows * B; i += stride) x[i] = z[i];
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->neg = 1;
      sc->done = 1;
    }
    return;
  }
  const double alpha = rz_old / pq;
  double rz = 0.0, rr = 0.0;
  for (long long row = (long long)blockIdx.x * kThreads + threadIdx.x; row < n_rows; row += stride) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const long long k = row * B + i;
      x[k] = fma(alpha, p[k], x[k]);
      r[k] = fma(-alpha, q[k], r[k]);
    }
    bj_apply_row<B>(inv, r, z, row);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      rz = fma(r[row * B + i], z[row * B + i], rz);
      rr = fma(r[row * B + i], r[row * B + i], rr);
    }
  }
  double s[2] = {block_sum(rz, sh), block_sum(rr, sh)};
  double out[2];
  if (finish_partials(partials, 2, s, ticket, out) && threadIdx.x == 0) {
    sc->beta = out[0] / rz_old;
    sc->rz = out[0];
    sc->rr = out[1];
    sc->iters += 1;
  }
}

template <int B>
__global__ void k_pcg_direction(const double* __restrict__ z, double* p, long long n, const PcgScalars* sc) {
  if (sc->done) return;
  const double beta = sc->beta;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

int grid_rows(long long n_rows, int rows_per_cta) {
  const long long g = (n_rows + rows_per_cta - 1) / rows_per_cta;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int bsr_spmv(int b, const int* row_ptr, const int* col_idx, const double* vals, const double* x, double* y,
             long long n_rows, double tau, SolverWork* w, double* dot_out, void* stream, PcgScalars* pcg) {
  cudaStream_t s = (cudaStream_t)stream;
  // b = 3: 8 lanes per block row (config 2: 15 blocks per row, ~2 per lane); measured on B200
  // 4 / 8 / 16 / 32 lanes: 72 / 83 / 75 / 50 % of the HBM roofline
  constexpr int G3 = 8;
  const int grid = grid_rows(n_rows, kThreads / (b == 3 ? G3 : 8));
  if (dot_out && grid > w->max_partials) return (int)cudaErrorInvalidValue;
  if (b == 3) {
    k_spmv<3, G3><<<grid, kThreads, 0, s>>>(row_ptr, col_idx, vals, x, y, n_rows, tau, w->partials, w->ticket, dot_out,
                                            pcg);
  } else if (b == 1) {
    constexpr int G = 8;
    k_spmv<1, G><<<grid, kThreads, 0, s>>>(row_ptr, col_idx, vals, x, y, n_rows, tau, w->partials, w->ticket, dot_out,
                                           pcg);
  } else {
    return (int)cudaErrorInvalidValue;
  }
  if (dot_out) k_sum_partials<<<1, kSumThreads, 0, s>>>(w->partials, grid, dot_out, pcg);
  return (int)cudaGetLastError();
}

long long spmv_partials_needed(int b, long long n_rows) {
  return grid_rows(n_rows, kThreads / 8);
}

int block_jacobi_inverse(int b, const int* row_ptr, const int* col_idx, const double* vals, long long n_rows,
                         double tau, double* inv, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_rows(n_rows, 128);
  if (b == 3) k_bj_inverse<3><<<grid, 128, 0, s>>>(row_ptr, col_idx, vals, n_rows, tau, inv);
  else if (b == 1) k_bj_inverse<1><<<grid, 128, 0, s>>>(row_ptr, col_idx, vals, n_rows, tau, inv);
  else return (int)cudaErrorInvalidValue;
  return (int)cudaGetLastError();
}

int pcg_init(int b, const double* rhs, SolverWork* w, long long n_rows, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = w->vec_grid;
  if (b == 3)
    k_pcg_init<3><<<grid, kThreads, 0, s>>>(rhs, w->inv, w->x, w->r, w->z, w->p, n_rows, w->partials, w->ticket, w->sc);
  else if (b == 1)
    k_pcg_init<1><<<grid, kThreads, 0, s>>>(rhs, w->inv, w->x, w->r, w->z, w->p, n_rows, w->partials, w->ticket, w->sc);
  else
    return (int)cudaErrorInvalidValue;
  return (int)cudaGetLastError();
}

int pcg_iteration(int b, const int* row_ptr, const int* col_idx, const double* vals, double tau, SolverWork* w,
                  long long n_rows, int it, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = bsr_spmv(b, row_ptr, col_idx, vals, w->p, w->q, n_rows, tau, w, &w->sc->pq, stream, w->sc);
  if (rc) return rc;
  const int grid = w->vec_grid;
  const long long n = n_rows * b;
  if (b == 3) {
    k_pcg_update<3><<<grid, kThreads, 0, s>>>(w->inv, w->x, w->r, w->z, w->p, w->q, n_rows, it, w->partials, w->ticket, w->sc);
    k_pcg_direction<3><<<grid, kThreads, 0, s>>>(w->z, w->p, n, w->sc);
  } else {
    k_pcg_update<1><<<grid, kThreads, 0, s>>>(w->inv, w->x, w->r, w->z, w->p, w->q, n_rows, it, w->partials, w->ticket, w->sc);
    k_pcg_direction<1><<<grid, kThreads, 0, s>>>(w->z, w->p, n, w->sc);
  }
  return (int)cudaGetLastError();
}

}  // namespace symel_cuda::dev
