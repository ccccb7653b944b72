// Static sm_100a kernels of the device assembly path (everything that is not generated
// from a tape): sparsity pattern + element->slot maps (replaces build_pattern,
// assembly.hpp:271-375), the reference-order scatter (assembly.hpp:450-462), energy sums and
// the finiteness reduction (assembly.hpp:426-448), activation compaction and guard minimum
// (assembly.hpp:143-173, 227-261), and pins (assembly.hpp:464-489).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <cstdlib>

#include <limits>
#include <vector>

#include "device_ops.hpp"

namespace symel_cuda::dev {

namespace {

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

template <class T>
int dalloc(T** p, size_t n, void* s) {
  return (int)cudaMallocAsync((void**)p, sizeof(T) * (n ? n : 1), S(s));
}

int bits_for(unsigned long long v) {
  int b = 1;
  while (b < 64 && (1ull << b) <= v) ++b;
  return b;
}

__device__ __forceinline__ long long lb_block(const LbDesc& d, const int* tup, int q) {
  return (d.off[q] + (long long)tup[d.slot[q]] * d.comps[q]) / d.b;
}

__global__ void k_pattern_keys(LbDesc d, const int* __restrict__ conn, const int* __restrict__ active,
                               long long n, unsigned long long* __restrict__ keys,
                               unsigned long long* counter) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long e = active ? active[t] : t;
  const int* tup = conn + e * d.arity;
  long long blk[kMaxLb];
  for (int q = 0; q < d.n_lb; ++q) blk[q] = lb_block(d, tup, q);
  int cnt = 0;
  for (int i = 0; i < d.n_lb; ++i)
    for (int j = 0; j < d.n_lb; ++j) cnt += blk[i] != blk[j];
  unsigned long long pos = atomicAdd(counter, (unsigned long long)cnt);
  for (int i = 0; i < d.n_lb; ++i)
    for (int j = 0; j < d.n_lb; ++j)
      if (blk[i] != blk[j]) keys[pos++] = ((unsigned long long)blk[i] << 32) | (unsigned long long)blk[j];
}

__global__ void k_diag_keys(long long n, unsigned long long* keys) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) keys[r] = ((unsigned long long)r << 32) | (unsigned long long)r;
}

__global__ void k_row_ptr(const unsigned long long* __restrict__ keys, long long nk, long long n_rows,
                          int* __restrict__ row_ptr, int* __restrict__ col_idx) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nk) {
    const unsigned long long k = keys[i];
    col_idx[i] = (int)(k & 0xffffffffull);
    const long long r = (long long)(k >> 32);
    const long long pr = i == 0 ? -1 : (long long)(keys[i - 1] >> 32);
    for (long long q = pr + 1; q <= r; ++q) row_ptr[q] = (int)i;  // rows start here
    if (i == nk - 1)
      for (long long q = r + 1; q <= n_rows; ++q) row_ptr[q] = (int)nk;
  }
}

__device__ __forceinline__ int find_block(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                                          long long r, long long c) {
  int lo = row_ptr[r], hi = row_ptr[r + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_slot_map(LbDesc d, const int* __restrict__ conn, const int* __restrict__ active, long long n,
                           const int* __restrict__ row_ptr, const int* __restrict__ col_idx, int* __restrict__ slots) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long e = active ? active[t] : t;
  const int* tup = conn + e * d.arity;
  long long blk[kMaxLb];
  for (int q = 0; q < d.n_lb; ++q) blk[q] = lb_block(d, tup, q);
  int* out = slots + t * d.n_lb * d.n_lb;
  for (int i = 0; i < d.n_lb; ++i)
    for (int j = 0; j < d.n_lb; ++j) out[i * d.n_lb + j] = find_block(row_ptr, col_idx, blk[i], blk[j]);
}

__global__ void k_refs(const int* __restrict__ slots, const int* __restrict__ conn, const int* __restrict__ active,
                       long long n, long long ord_base, LbDesc d, unsigned long long pos_h, unsigned long long pos_g,
                       unsigned* __restrict__ hkey, unsigned long long* __restrict__ hval, unsigned* __restrict__ gkey,
                       unsigned long long* __restrict__ gval) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long e = active ? active[t] : t;
  const int* tup = conn + e * d.arity;
  const int nl = d.n_lb;
  const unsigned long long ord = (unsigned long long)(ord_base + t);
  for (int i = 0; i < nl; ++i) {
    gkey[pos_g + t * nl + i] = (unsigned)lb_block(d, tup, i);
    gval[pos_g + t * nl + i] = (ord << 5) | (unsigned long long)i;
    for (int j = 0; j < nl; ++j) {
      const long long q = pos_h + (t * nl + i) * nl + j;
      hkey[q] = (unsigned)slots[(t * nl + i) * nl + j];
      hval[q] = (ord << 10) | ((unsigned long long)i << 5) | (unsigned long long)j;
    }
  }
}

__global__ void k_seg_ptr(const unsigned* __restrict__ keys, long long nk, long long nseg, int* __restrict__ ptr) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nk) {
    const long long r = keys[i];
    const long long pr = i == 0 ? -1 : (long long)keys[i - 1];
    for (long long q = pr + 1; q <= r; ++q) ptr[q] = (int)i;
    if (i == nk - 1)
      for (long long q = r + 1; q <= nseg; ++q) ptr[q] = (int)nk;
  }
  if (nk == 0 && i <= nseg) ptr[i] = 0;
}

struct LayoutTable {
  ContribLayout e[8];
  int n;
};

__device__ __forceinline__ const ContribLayout& which(const LayoutTable& L, unsigned long long ord) {
  int k = 0;
  while (k + 1 < L.n && (long long)ord >= L.e[k].ord_end) ++k;
  return L.e[k];
}

// One thread per BSR block: contributions in ascending (energy, element, a, c) order from +0.0.
__global__ void k_ordered_hess(LayoutTable L, const int* __restrict__ ptr, const unsigned long long* __restrict__ ref,
                               long long n_blocks, int b, double* __restrict__ vals) {
  const long long blk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= n_blocks) return;
  double acc[9];
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  for (int k = ptr[blk]; k < ptr[blk + 1]; ++k) {
    const unsigned long long r = ref[k];
    const unsigned long long ord = r >> 10;
    const int li = (int)((r >> 5) & 31), lj = (int)(r & 31);
    const ContribLayout& c = which(L, ord);
    const double* src = c.contrib + (long long)(ord - c.ord_base) * c.stride + 1 + c.n_dofs;
    for (int ri = 0; ri < b; ++ri) {
      const int di = c.dof_of[li * 3 + ri];
      if (di < 0) continue;
      for (int rj = 0; rj < b; ++rj) {
        const int dj = c.dof_of[lj * 3 + rj];
        if (dj < 0) continue;
        acc[ri * b + rj] += src[di * c.n_dofs + dj];
      }
    }
  }
  for (int q = 0; q < b * b; ++q) vals[blk * b * b + q] = acc[q];
}

__global__ void k_ordered_grad(LayoutTable L, const int* __restrict__ ptr, const unsigned long long* __restrict__ ref,
                               long long n_rows, int b, double* __restrict__ grad) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n_rows) return;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int k = ptr[row]; k < ptr[row + 1]; ++k) {
    const unsigned long long r = ref[k];
    const unsigned long long ord = r >> 5;
    const int li = (int)(r & 31);
    const ContribLayout& c = which(L, ord);
    const double* src = c.contrib + (long long)(ord - c.ord_base) * c.stride + 1;
    for (int q = 0; q < b; ++q) {
      const int d = c.dof_of[li * 3 + q];
      if (d >= 0) acc[q] += src[d];
    }
  }
  for (int q = 0; q < b; ++q) grad[row * b + q] = acc[q];
}

__global__ void k_gather_strided(const double* __restrict__ src, long long stride, long long n, double* __restrict__ dst) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i * stride];
}

__global__ void k_serial_sum(const double* __restrict__ v, long long n, double init_from, double* out, int accumulate) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double e = accumulate ? *out : 0.0;
  for (long long i = 0; i < n; ++i) e += v[i];
  *out = e;
  (void)init_from;
}

constexpr int kTreeChunk = 4096;  // fixed reduction shape => result independent of launch size
constexpr int kTreeThreads = 256;

__global__ void k_tree_partial(const double* __restrict__ v, long long stride, long long n, double* __restrict__ partial) {
  __shared__ double sh[kTreeThreads];
  const long long base = (long long)blockIdx.x * kTreeChunk;
  double s = 0.0;
  for (int q = 0; q < kTreeChunk / kTreeThreads; ++q) {
    const long long i = base + (long long)q * kTreeThreads + threadIdx.x;
    if (i < n) s += v[i * stride];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kTreeThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_tree_final(const double* __restrict__ partial, long long n, double* out) {
  __shared__ double sh[kTreeThreads];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += kTreeThreads) s += partial[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kTreeThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void k_combine(const double* __restrict__ v, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double e = 0.0;
    for (int i = 0; i < n; ++i) e += v[i];
    *out = e;
  }
}

__global__ void k_act_mask(const double* __restrict__ v, long long n, int kind, unsigned char* __restrict__ mask,
                           int* changed) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = v[i];
  const unsigned char a = kind == 0 ? (x >= 0.0) : (x > 0.0);  // Condition::holds, expr.hpp:574
  if (a != mask[i]) {
    mask[i] = a;
    *changed = 1;
  }
}

struct MinOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return b < a ? b : a; }
};

__global__ void k_pins(const unsigned char* __restrict__ mask, long long n_rows, int b, const int* __restrict__ row_ptr,
                       const int* __restrict__ col_idx, double* __restrict__ vals, double* __restrict__ grad) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  for (int q = 0; q < b; ++q)
    if (mask[r * b + q]) grad[r * b + q] = 0.0;
  for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
    const long long c = col_idx[k];
    double* v = vals + (long long)k * b * b;
    for (int i = 0; i < b; ++i) {
      const bool pr = mask[r * b + i] != 0;
      for (int j = 0; j < b; ++j)
        if (pr || mask[c * b + j]) v[i * b + j] = 0.0;
    }
    if (c == r)
      for (int i = 0; i < b; ++i)
        if (mask[r * b + i]) v[i * b + i] = 1.0;
  }
}

inline unsigned grid_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// FP64 pipe peak probe: 8 independent DFMA chains per thread (enough ILP for full issue).
__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double b, double c, double* sink) {
  double a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9 + q;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
  double s = 0;
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 123.456) *sink = s;
}

}  // namespace

int fp64_peak(int n_sm, double* tflops, void* s) {
  double* sink;
  int err;
  if ((err = dalloc(&sink, 1, s))) return err;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 14, blocks = n_sm * 8, threads = 256;
  k_dfma_peak<<<blocks, threads, 0, S(s)>>>(64, 0.999999, 1e-7, sink);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, S(s));
    k_dfma_peak<<<blocks, threads, 0, S(s)>>>(iters, 0.999999, 1e-7, sink);
    cudaEventRecord(e1, S(s));
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  *tflops = 2.0 * 8.0 * iters * (double)blocks * threads / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, S(s));
  return (int)cudaGetLastError();
}

int pattern_keys(const LbDesc& d, const int* conn, const int* active, long long n, unsigned long long* keys,
                 unsigned long long* counter, void* s) {
  if (n <= 0) return 0;
  k_pattern_keys<<<grid_for(n, 256), 256, 0, S(s)>>>(d, conn, active, n, keys, counter);
  return (int)cudaGetLastError();
}

int diag_keys(long long n_rows, unsigned long long* keys, void* s) {
  if (n_rows <= 0) return 0;
  k_diag_keys<<<grid_for(n_rows, 256), 256, 0, S(s)>>>(n_rows, keys);
  return (int)cudaGetLastError();
}

int build_csr(unsigned long long* keys, long long nk, long long n_rows, int** row_ptr, int** col_idx,
              long long* n_blocks, void* s) {
  int err;
  unsigned long long* sorted = nullptr;
  if ((err = dalloc(&sorted, nk, s))) return err;
  const int end_bit = 32 + bits_for((unsigned long long)n_rows);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, sorted, nk, 0, end_bit, S(s));
  void* tmp = nullptr;
  if ((err = dalloc((char**)&tmp, tmp_bytes, s))) return err;
  cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, nk, 0, end_bit, S(s));
  cudaFreeAsync(tmp, S(s));
  long long* d_nu = nullptr;
  if ((err = dalloc(&d_nu, 1, s))) return err;
  tmp_bytes = 0;
  cub::DeviceSelect::Unique(nullptr, tmp_bytes, sorted, keys, d_nu, nk, S(s));
  if ((err = dalloc((char**)&tmp, tmp_bytes, s))) return err;
  cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, keys, d_nu, nk, S(s));
  cudaFreeAsync(tmp, S(s));
  cudaFreeAsync(sorted, S(s));
  long long nu = 0;
  cudaMemcpyAsync(&nu, d_nu, sizeof nu, cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  cudaFreeAsync(d_nu, S(s));
  if (nu >= (1ll << 31)) return (int)cudaErrorInvalidValue;
  if ((err = dalloc(row_ptr, n_rows + 1, s))) return err;
  if ((err = dalloc(col_idx, nu, s))) return err;
  k_row_ptr<<<grid_for(nu, 256), 256, 0, S(s)>>>(keys, nu, n_rows, *row_ptr, *col_idx);
  *n_blocks = nu;
  return (int)cudaGetLastError();
}

int slot_map(const LbDesc& d, const int* conn, const int* active, long long n, const int* row_ptr,
             const int* col_idx, int* slots, void* s) {
  if (n <= 0) return 0;
  k_slot_map<<<grid_for(n, 128), 128, 0, S(s)>>>(d, conn, active, n, row_ptr, col_idx, slots);
  return (int)cudaGetLastError();
}

int ordered_refs(const EnergyRefSrc* src, int ne, long long n_blocks, long long n_rows, OrderedRefs* out,
                 void* s) {
  int err;
  long long nh = 0, ng = 0;
  for (int k = 0; k < ne; ++k) {
    nh += src[k].n_active * src[k].d.n_lb * src[k].d.n_lb;
    ng += src[k].n_active * src[k].d.n_lb;
  }
  unsigned *hk, *gk, *hk2, *gk2;
  unsigned long long *hv, *gv, *hv2, *gv2;
  if ((err = dalloc(&hk, nh, s)) || (err = dalloc(&hv, nh, s)) || (err = dalloc(&gk, ng, s)) ||
      (err = dalloc(&gv, ng, s)) || (err = dalloc(&hk2, nh, s)) || (err = dalloc(&hv2, nh, s)) ||
      (err = dalloc(&gk2, ng, s)) || (err = dalloc(&gv2, ng, s)))
    return err;
  unsigned long long ph = 0, pg = 0;
  for (int k = 0; k < ne; ++k) {
    const EnergyRefSrc& e = src[k];
    if (e.n_active > 0)
      k_refs<<<grid_for(e.n_active, 128), 128, 0, S(s)>>>(e.slots, e.conn, e.active, e.n_active, e.ord_base, e.d,
                                                          ph, pg, hk, hv, gk, gv);
    ph += (unsigned long long)e.n_active * e.d.n_lb * e.d.n_lb;
    pg += (unsigned long long)e.n_active * e.d.n_lb;
  }
  // stable LSD radix sort keeps the generation order (energy, element, a, c) per key
  size_t tb = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, hk, hk2, hv, hv2, nh, 0, bits_for(n_blocks), S(s));
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, gk, gk2, gv, gv2, ng, 0, bits_for(n_rows), S(s));
  void* tmp;
  if ((err = dalloc((char**)&tmp, tb > tb2 ? tb : tb2, s))) return err;
  cub::DeviceRadixSort::SortPairs(tmp, tb, hk, hk2, hv, hv2, nh, 0, bits_for(n_blocks), S(s));
  tb2 = tb > tb2 ? tb : tb2;
  cub::DeviceRadixSort::SortPairs(tmp, tb2, gk, gk2, gv, gv2, ng, 0, bits_for(n_rows), S(s));
  cudaFreeAsync(tmp, S(s));
  if ((err = dalloc(&out->hess_ptr, n_blocks + 1, s)) || (err = dalloc(&out->grad_ptr, n_rows + 1, s))) return err;
  k_seg_ptr<<<grid_for(nh > n_blocks + 1 ? nh : n_blocks + 1, 256), 256, 0, S(s)>>>(hk2, nh, n_blocks, out->hess_ptr);
  k_seg_ptr<<<grid_for(ng > n_rows + 1 ? ng : n_rows + 1, 256), 256, 0, S(s)>>>(gk2, ng, n_rows, out->grad_ptr);
  cudaFreeAsync(hk, S(s)); cudaFreeAsync(hv, S(s)); cudaFreeAsync(gk, S(s)); cudaFreeAsync(gv, S(s));
  cudaFreeAsync(hk2, S(s)); cudaFreeAsync(gk2, S(s));
  out->hess_ref = hv2;
  out->grad_ref = gv2;
  out->n_hess = nh;
  out->n_grad = ng;
  return (int)cudaGetLastError();
}

void free_ordered_refs(OrderedRefs* r) {
  cudaFree(r->hess_ptr); cudaFree(r->hess_ref); cudaFree(r->grad_ptr); cudaFree(r->grad_ref);
  *r = OrderedRefs{};
}

int ordered_scatter(const ContribLayout* lay, int ne, const OrderedRefs& r, long long n_blocks, long long n_rows,
                    double* vals, double* grad, void* s) {
  if (ne > 8) return (int)cudaErrorInvalidValue;
  LayoutTable L{};
  L.n = ne;
  for (int k = 0; k < ne; ++k) L.e[k] = lay[k];
  const int b = lay[0].b;
  if (n_blocks > 0) k_ordered_hess<<<grid_for(n_blocks, 128), 128, 0, S(s)>>>(L, r.hess_ptr, r.hess_ref, n_blocks, b, vals);
  if (n_rows > 0) k_ordered_grad<<<grid_for(n_rows, 128), 128, 0, S(s)>>>(L, r.grad_ptr, r.grad_ref, n_rows, b, grad);
  return (int)cudaGetLastError();
}

int energy_serial(const double* const* elemE, const long long* strides, const long long* counts, int ne,
                  double* out, void* s) {
  long long mx = 0;
  for (int k = 0; k < ne; ++k) mx = counts[k] > mx ? counts[k] : mx;
  double* tmp;
  int err;
  if ((err = dalloc(&tmp, mx, s))) return err;
  cudaMemsetAsync(out, 0, sizeof(double), S(s));
  for (int k = 0; k < ne; ++k) {
    if (counts[k] == 0) continue;
    k_gather_strided<<<grid_for(counts[k], 256), 256, 0, S(s)>>>(elemE[k], strides[k], counts[k], tmp);
    k_serial_sum<<<1, 32, 0, S(s)>>>(tmp, counts[k], 0.0, out, 1);
  }
  cudaFreeAsync(tmp, S(s));
  return (int)cudaGetLastError();
}

int energy_tree(const double* v, long long stride, long long n, double* partial, double* out, void* s) {
  if (n == 0) return (int)cudaMemsetAsync(out, 0, sizeof(double), S(s));
  const long long nb = (n + kTreeChunk - 1) / kTreeChunk;
  if (nb == 1) {  // one chunk: its tree sum is the result (the final pass would only add zeros to it)
    k_tree_partial<<<1, kTreeThreads, 0, S(s)>>>(v, stride, n, out);
    return (int)cudaGetLastError();
  }
  k_tree_partial<<<(unsigned)nb, kTreeThreads, 0, S(s)>>>(v, stride, n, partial);
  k_tree_final<<<1, kTreeThreads, 0, S(s)>>>(partial, nb, out);
  return (int)cudaGetLastError();
}

long long energy_tree_partials(long long n) { return (n + kTreeChunk - 1) / kTreeChunk; }
int energy_tree_launches(long long n) { return n <= 0 ? 0 : (n <= kTreeChunk ? 1 : 2); }

int energy_combine(const double* per_energy, int n, double* out, void* s) {
  k_combine<<<1, 32, 0, S(s)>>>(per_energy, n, out);
  return (int)cudaGetLastError();
}

int activation_mask(const double* v, long long n, int kind, unsigned char* mask, int* changed, void* s) {
  if (n <= 0) return 0;
  k_act_mask<<<grid_for(n, 256), 256, 0, S(s)>>>(v, n, kind, mask, changed);
  return (int)cudaGetLastError();
}

int compact_active(const unsigned char* mask, long long n, int* active, long long* n_active_host, void* s) {
  int err;
  long long* d_n;
  if ((err = dalloc(&d_n, 1, s))) return err;
  size_t tb = 0;
  cub::CountingInputIterator<int> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb, it, mask, active, d_n, n, S(s));
  void* tmp;
  if ((err = dalloc((char**)&tmp, tb, s))) return err;
  cub::DeviceSelect::Flagged(tmp, tb, it, mask, active, d_n, n, S(s));
  cudaMemcpyAsync(n_active_host, d_n, sizeof(long long), cudaMemcpyDeviceToHost, S(s));
  cudaFreeAsync(tmp, S(s));
  cudaFreeAsync(d_n, S(s));
  return (int)cudaStreamSynchronize(S(s));
}

int min_reduce(const double* v, long long n, double* out, void* s) {
  size_t tb = 0;
  cub::DeviceReduce::Reduce(nullptr, tb, v, out, n, MinOp(), std::numeric_limits<double>::infinity(), S(s));
  void* tmp;
  int err;
  if ((err = dalloc((char**)&tmp, tb, s))) return err;
  cub::DeviceReduce::Reduce(tmp, tb, v, out, n, MinOp(), std::numeric_limits<double>::infinity(), S(s));
  cudaFreeAsync(tmp, S(s));
  return (int)cudaGetLastError();
}

int apply_pins(const unsigned char* mask, long long n_rows, int b, const int* row_ptr, const int* col_idx,
               double* vals, double* grad, void* s) {
  if (n_rows <= 0) return 0;
  k_pins<<<grid_for(n_rows, 128), 128, 0, S(s)>>>(mask, n_rows, b, row_ptr, col_idx, vals, grad);
  return (int)cudaGetLastError();
}

// =================================================================== tile plan (K3)

namespace {

// Hessian, upper BSR blocks only: each unordered local pair {i, j} contributes to the block
// (min(gi, gj), max(gi, gj)) as the element sub-block (row side, col side); equal global blocks
// from distinct local blocks (a repeated node) contribute both orientations to the diagonal.
// key (global tile << 32 | block), value (position-in-tile << 10 | li << 5 | lj); unused
// key slots hold `sentinel` and sort last.
__global__ void k_tile_hkeys(TileSrc src, unsigned long long pos, unsigned long long sentinel,
                             unsigned long long* keys, unsigned short* vals) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= src.n_active) return;
  const long long t = src.perm ? src.perm[p] : p;  // active ordinal at this tile position
  const long long e = src.active ? src.active[t] : t;
  const int* tup = src.conn + e * src.d.arity;
  const int nl = src.d.n_lb;
  long long g[kMaxLb];
  for (int q = 0; q < nl; ++q) g[q] = lb_block(src.d, tup, q);
  const unsigned long long tile = (unsigned long long)(src.tile_base + p / src.tpb);
  const unsigned tl = (unsigned)(p % src.tpb);
  const int* sl = src.slots + t * nl * nl;
  long long q = pos + p * nl * nl;
  auto put = [&](int li, int lj) {
    const int lo = li < lj ? li : lj, hi = li < lj ? lj : li;
    const unsigned sub = (unsigned)(lo * nl - ((lo * (lo - 1)) >> 1) + (hi - lo));
    keys[q] = (tile << 32) | (unsigned)sl[li * nl + lj];
    vals[q] = (unsigned short)(((li > lj) ? 0x8000u : 0u) | (sub << 7) | tl);
    ++q;
  };
  for (int i = 0; i < nl; ++i)
    for (int j = i; j < nl; ++j) {
      if (g[i] < g[j]) put(i, j);
      else if (g[i] > g[j]) put(j, i);
      else {
        put(i, j);
        if (i != j) put(j, i);
      }
    }
  for (const long long q1 = pos + (p + 1) * nl * nl; q < q1; ++q) {
    keys[q] = sentinel;
    vals[q] = 0;
  }
}

// gradient: key (global tile << 32 | block row), value (position-in-tile << 5 | li)
__global__ void k_tile_gkeys(TileSrc src, unsigned long long pos, unsigned long long* keys, unsigned short* vals) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= src.n_active) return;
  const long long t = src.perm ? src.perm[p] : p;
  const long long e = src.active ? src.active[t] : t;
  const int* tup = src.conn + e * src.d.arity;
  const int nl = src.d.n_lb;
  const unsigned long long tile = (unsigned long long)(src.tile_base + p / src.tpb);
  const unsigned tl = (unsigned)(p % src.tpb);
  for (int i = 0; i < nl; ++i) {
    keys[pos + p * nl + i] = (tile << 32) | (unsigned)lb_block(src.d, tup, i);
    vals[pos + p * nl + i] = (unsigned short)(((unsigned)i << 7) | tl);
  }
}

// mirror (transposed) block of each segment's target block
__global__ void k_seg_mirror(const int* __restrict__ target, long long n, const int* __restrict__ row_ptr,
                             long long n_rows, const int* __restrict__ col_idx, int* __restrict__ mirror,
                             unsigned char* __restrict__ touched) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = target[i];
  long long lo = 0, hi = n_rows;  // row r: row_ptr[r] <= b < row_ptr[r + 1]
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= b) lo = mid; else hi = mid;
  }
  const int m = find_block(row_ptr, col_idx, col_idx[b], lo);
  mirror[i] = m;
  touched[b] = 1;
  touched[m] = 1;
}

// Morton code of an element's centroid (first three components of its local-block items)
__device__ __forceinline__ unsigned spread10(unsigned v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void k_centroids(LbDesc d, const double* const* arrs, const int* __restrict__ conn,
                            const int* __restrict__ active, long long n, double* __restrict__ cen) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long e = active ? active[t] : t;
  const int* tup = conn + e * d.arity;
  double c[3] = {0, 0, 0};
  for (int q = 0; q < d.n_lb; ++q) {
    const double* p = arrs[q] + (long long)tup[d.slot[q]] * d.comps[q];
    for (int k = 0; k < 3 && k < d.comps[q]; ++k) c[k] += p[k];
  }
  for (int k = 0; k < 3; ++k) cen[3 * t + k] = c[k] / d.n_lb;
}

__global__ void k_morton_keys(const double* __restrict__ cen, long long n, double3 lo, double3 inv,
                              unsigned* __restrict__ key, int* __restrict__ ord) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  auto qz = [](double v) { return (unsigned)fmin(1023.0, fmax(0.0, v)); };
  key[t] = spread10(qz((cen[3 * t] - lo.x) * inv.x)) | (spread10(qz((cen[3 * t + 1] - lo.y) * inv.y)) << 1) |
           (spread10(qz((cen[3 * t + 2] - lo.z) * inv.z)) << 2);
  ord[t] = (int)t;
}

__global__ void k_compose(const int* __restrict__ perm, const int* __restrict__ active, long long n, int* __restrict__ elems) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) elems[p] = active ? active[perm[p]] : perm[p];
}

__global__ void k_not(const unsigned char* __restrict__ a, long long n, unsigned char* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = !a[i];
}

__global__ void k_split_keys(const unsigned long long* __restrict__ ukeys, long long n, int* __restrict__ seg_tile,
                             int* __restrict__ seg_target) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  seg_tile[i] = (int)(ukeys[i] >> 32);
  seg_target[i] = (int)(ukeys[i] & 0xffffffffull);
}

__global__ void k_tile_max(const int* __restrict__ tile_seg_ptr, const int* __restrict__ seg_con_ptr, long long n_tiles,
                           int* mx, int* __restrict__ tile_con_ptr) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  const int s0 = tile_seg_ptr[t];
  tile_con_ptr[t] = seg_con_ptr[s0];
  if (t == n_tiles) return;
  const int s1 = tile_seg_ptr[t + 1];
  atomicMax(mx, s1 - s0);
  atomicMax(mx + 1, seg_con_ptr[s1] - seg_con_ptr[s0]);
}

// segment sort key: tile-major, contribution count descending (stable: target order on ties)
__global__ void k_seg_sort_keys(const unsigned long long* __restrict__ ukeys, const int* __restrict__ counts,
                                const unsigned char* __restrict__ tile_sort, long long n,
                                unsigned long long* __restrict__ key, int* __restrict__ idx) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long tile = ukeys[i] >> 32;
  key[i] = (tile << 32) | (tile_sort[tile] ? (unsigned long long)(0xffffffffu - (unsigned)counts[i]) : 0ull);
  idx[i] = (int)i;
}

__global__ void k_seg_permute(const int* __restrict__ perm, const unsigned long long* __restrict__ ukeys,
                              const int* __restrict__ counts, long long n, unsigned long long* __restrict__ ukeys2,
                              int* __restrict__ counts2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ukeys2[i] = ukeys[perm[i]];
  counts2[i] = counts[perm[i]];
}

__global__ void k_con_permute(const int* __restrict__ perm, const int* __restrict__ old_ptr,
                              const int* __restrict__ new_ptr, long long n, const unsigned short* __restrict__ con,
                              unsigned short* __restrict__ con2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int o = old_ptr[perm[i]], d = new_ptr[i], c = new_ptr[i + 1] - d;
  for (int k = 0; k < c; ++k) con2[d + k] = con[o + k];
}

// per segment: its first contribution relative to its tile's first (16 bits: <= 65535 per tile)
__global__ void k_seg_rel(const int* __restrict__ seg_tile, const int* __restrict__ seg_con_ptr,
                          const int* __restrict__ tile_con_ptr, long long n, unsigned short* __restrict__ rel) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rel[i] = (unsigned short)(seg_con_ptr[i] - tile_con_ptr[seg_tile[i]]);
}

__global__ void k_count_targets(const int* __restrict__ seg_target, long long n, int* __restrict__ count) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(count + seg_target[i], 1);
}

// over segments sorted by (target, tile): flag boundary segments
__global__ void k_boundary_flags(const int* __restrict__ sorted_target, long long n, const int* __restrict__ count,
                                 int* __restrict__ flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = count[sorted_target[i]] > 1;
}

__global__ void k_seg_dst(const int* __restrict__ sorted_target, const int* __restrict__ sorted_seg,
                          const int* __restrict__ flag, const int* __restrict__ pos, long long n, int* __restrict__ seg_dst) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  seg_dst[sorted_seg[i]] = flag[i] ? -(pos[i] + 1) : sorted_target[i];
}

__global__ void k_iota(int* v, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int)i;
}

__global__ void k_is_zero(const int* __restrict__ count, long long n, unsigned char* __restrict__ flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = count[i] == 0;
}

// sorted int keys -> ptr[k] = first index with key >= k, for k in [0, nseg]
__global__ void k_int_seg_ptr(const int* __restrict__ keys, long long nk, long long nseg, int* __restrict__ ptr) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nk) {
    const long long r = keys[i];
    const long long pr = i == 0 ? -1 : (long long)keys[i - 1];
    for (long long q = pr + 1; q <= r; ++q) ptr[q] = (int)i;
    if (i == nk - 1)
      for (long long q = r + 1; q <= nseg; ++q) ptr[q] = (int)nk;
  }
  if (nk == 0 && i <= nseg) ptr[i] = 0;
}

// One thread per (shared target, entry): partials of the target in (energy, tile) order; a
// Hessian target also writes the transposed entry of its mirror (lower) block.
__global__ void k_fixup(const int* __restrict__ pt_ptr, const int* __restrict__ pt_target, const int* __restrict__ mirror,
                        long long n_pt, int w, int b, const double* __restrict__ partials, double* __restrict__ out) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_pt * w) return;
  const long long p = q / w;
  const int ent = (int)(q % w);
  const int k0 = __ldg(pt_ptr + p), k1 = __ldg(pt_ptr + p + 1);
  const int tg = __ldg(pt_target + p), mr = mirror ? __ldg(mirror + p) : tg;
  // partials in slot order, summed left to right from +0.0. The first kFixIlp are loaded
  // predicated, all at once: one memory round trip after the index loads instead of one per
  // partial (targets have ~2.6 (config 2) to ~7 (config 4) partials; rows up to ~13)
  constexpr int kFixIlp = 16;
  const int n = k1 - k0;
  double v[kFixIlp];
#pragma unroll
  for (int i = 0; i < kFixIlp; ++i) v[i] = i < n ? __ldcs(partials + (long long)(k0 + i) * w + ent) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < kFixIlp; ++i)
    if (i < n) acc += v[i];
  for (int k = k0 + kFixIlp; k < k1; ++k) acc += __ldcs(partials + (long long)k * w + ent);
  out[(long long)tg * w + ent] = acc;
  if (mr != tg) out[(long long)mr * w + (ent % b) * b + ent / b] = acc;
}

// The same fix-up with the entry count W (b*b or b) and block size B compile-time and 32-bit
// thread indices (q / W by a constant): the generic kernel's 64-bit division by a runtime
// width and its 16 predicated loads made it issue-bound (366 instructions per warp, 48 % of
// HBM at config 2). Same summation: partials in slot order, left to right from +0.0. The first
// four partials (config 2: 2.6 per target on average) are loaded at once.
template <int W, int B>
__global__ void __launch_bounds__(256) k_fixup_w(const int* __restrict__ pt_ptr, const int* __restrict__ pt_target,
                                                 const int* __restrict__ mirror, unsigned n_pt,
                                                 const double* __restrict__ partials, double* __restrict__ out) {
  const unsigned q = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned p = q / W, ent = q - p * W;
  if (p >= n_pt) return;
  const int k0 = __ldg(pt_ptr + p), k1 = __ldg(pt_ptr + p + 1);
  const int tg = __ldg(pt_target + p);
  const int mr = mirror ? __ldg(mirror + p) : tg;
  const double* src = partials + (size_t)k0 * W + ent;
  const int n = k1 - k0;
  double v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = i < n ? __ldcs(src + i * W) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < n) acc += v[i];
  for (int k = 4; k < n; ++k) acc += __ldcs(src + (size_t)k * W);
  out[(size_t)tg * W + ent] = acc;
  if (W == B * B && mr != tg) out[(size_t)mr * W + (ent % B) * B + ent / B] = acc;
}

template <int B>
bool fixup_fast(const SegPlan& sp, bool hess, const double* partials, double* out, cudaStream_t st) {
  constexpr int W2 = B * B;
  const long long w = hess ? W2 : B;
  if (sp.n_pt * w >= (1ll << 31)) return false;
  const unsigned nt = (unsigned)sp.n_pt;
  if (hess)
    k_fixup_w<W2, B><<<grid_for(sp.n_pt * w, 256), 256, 0, st>>>(sp.pt_ptr, sp.pt_target, sp.pt_mirror, nt, partials, out);
  else
    k_fixup_w<B, B><<<grid_for(sp.n_pt * w, 256), 256, 0, st>>>(sp.pt_ptr, sp.pt_target, nullptr, nt, partials, out);
  return true;
}

bool fixup_dispatch(const SegPlan& sp, bool hess, int b, const double* partials, double* out, cudaStream_t st) {
  switch (b) {
    case 1: return fixup_fast<1>(sp, hess, partials, out, st);
    case 2: return fixup_fast<2>(sp, hess, partials, out, st);
    case 3: return fixup_fast<3>(sp, hess, partials, out, st);
    default: return false;
  }
}

__global__ void k_zero_targets(const int* __restrict__ tg, long long n, int w, double* __restrict__ out) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n * w) out[(long long)tg[q / w] * w + (q % w)] = 0.0;
}

template <class T>
int tmp_alloc(T** p, size_t n, void* s) {
  return (int)cudaMallocAsync((void**)p, sizeof(T) * (n ? n : 1), S(s));
}

// Sorts (key, val) and segments it; fills the common part of a SegPlan.
unsigned long long key_sentinel(long long n_tiles) {
  return (1ull << (32 + bits_for((unsigned long long)n_tiles))) - 1ull;
}

int build_segments(unsigned long long* keys, unsigned short* vals, long long n, long long n_tiles, long long n_targets,
                   const int* row_ptr, const int* col_idx, long long n_rows, const unsigned char* tile_sort,
                   SegPlan* sp, void* s) {
  int err;
  unsigned long long* k2;
  unsigned short* v2;
  if ((err = tmp_alloc(&k2, n, s)) || (err = tmp_alloc(&v2, n + 2, s))) return err;
  const int end_bit = 32 + bits_for((unsigned long long)n_tiles);
  const unsigned long long sentinel = key_sentinel(n_tiles);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, k2, vals, v2, n, 0, end_bit, S(s));
  void* tmp;
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceRadixSort::SortPairs(tmp, tb, keys, k2, vals, v2, n, 0, end_bit, S(s));  // stable: element order kept
  cudaFreeAsync(tmp, S(s));
  sp->con = v2;
  sp->n_con = n;
  // run-length encode (tile, target) -> segments
  unsigned long long* ukeys;
  int* counts;
  long long* d_nseg;
  if ((err = tmp_alloc(&ukeys, n, s)) || (err = tmp_alloc(&counts, n + 1, s)) || (err = tmp_alloc(&d_nseg, 1, s))) return err;
  tb = 0;
  cub::DeviceRunLengthEncode::Encode(nullptr, tb, k2, ukeys, counts, d_nseg, n, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceRunLengthEncode::Encode(tmp, tb, k2, ukeys, counts, d_nseg, n, S(s));
  cudaFreeAsync(tmp, S(s));
  long long nseg = 0;
  cudaMemcpyAsync(&nseg, d_nseg, sizeof nseg, cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  if (nseg > 0) {  // unused key slots (sentinel) form the last run: drop it
    unsigned long long last = 0;
    cudaMemcpyAsync(&last, ukeys + nseg - 1, sizeof last, cudaMemcpyDeviceToHost, S(s));
    if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
    if (last == sentinel) --nseg;
  }
  sp->n_seg = nseg;
  // Within each tile, order the segments by contribution count (descending, stable): the
  // threads of a warp then reduce segments of similar length (less divergence). Tiles stay
  // in order, so partials keep their (energy, tile) summation order.
  if (nseg > 1 && tile_sort && !std::getenv("SYMEL_NO_SEG_SORT")) {
    unsigned long long *skey, *skey2, *ukeys2;
    int *sidx, *sidx2, *counts2, *old_ptr, *new_ptr;
    unsigned short* con2;
    if ((err = tmp_alloc(&skey, nseg, s)) || (err = tmp_alloc(&skey2, nseg, s)) || (err = tmp_alloc(&ukeys2, nseg, s)) ||
        (err = tmp_alloc(&sidx, nseg, s)) || (err = tmp_alloc(&sidx2, nseg, s)) ||
        (err = tmp_alloc(&counts2, nseg + 1, s)) || (err = tmp_alloc(&old_ptr, nseg + 1, s)) ||
        (err = tmp_alloc(&new_ptr, nseg + 1, s)) || (err = tmp_alloc(&con2, n + 2, s)))
      return err;
    k_seg_sort_keys<<<grid_for(nseg, 256), 256, 0, S(s)>>>(ukeys, counts, tile_sort, nseg, skey, sidx);
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, skey, skey2, sidx, sidx2, nseg, 0, end_bit, S(s));
    if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
    cub::DeviceRadixSort::SortPairs(tmp, tb, skey, skey2, sidx, sidx2, nseg, 0, end_bit, S(s));
    cudaFreeAsync(tmp, S(s));
    k_seg_permute<<<grid_for(nseg, 256), 256, 0, S(s)>>>(sidx2, ukeys, counts, nseg, ukeys2, counts2);
    cudaMemsetAsync(counts + nseg, 0, sizeof(int), S(s));
    cudaMemsetAsync(counts2 + nseg, 0, sizeof(int), S(s));
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, old_ptr, nseg + 1, S(s));
    if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts, old_ptr, nseg + 1, S(s));
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts2, new_ptr, nseg + 1, S(s));
    cudaFreeAsync(tmp, S(s));
    k_con_permute<<<grid_for(nseg, 256), 256, 0, S(s)>>>(sidx2, old_ptr, new_ptr, nseg, v2, con2);
    cudaMemcpyAsync(ukeys, ukeys2, sizeof(unsigned long long) * nseg, cudaMemcpyDeviceToDevice, S(s));
    cudaMemcpyAsync(counts, counts2, sizeof(int) * nseg, cudaMemcpyDeviceToDevice, S(s));
    cudaMemcpyAsync(v2, con2, sizeof(unsigned short) * n, cudaMemcpyDeviceToDevice, S(s));
    for (void* q : {(void*)skey, (void*)skey2, (void*)ukeys2, (void*)sidx, (void*)sidx2, (void*)counts2, (void*)old_ptr,
                    (void*)new_ptr, (void*)con2})
      cudaFreeAsync(q, S(s));
  }
  // segment -> contribution ranges
  if ((err = tmp_alloc(&sp->seg_con_ptr, nseg + 1, s))) return err;
  cudaMemsetAsync(sp->seg_con_ptr + nseg, 0, sizeof(int), S(s));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, sp->seg_con_ptr, nseg + 1, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cudaMemsetAsync(counts + nseg, 0, sizeof(int), S(s));  // counts has >= nseg + 1 slots when n > nseg
  cub::DeviceScan::ExclusiveSum(tmp, tb, counts, sp->seg_con_ptr, nseg + 1, S(s));
  cudaFreeAsync(tmp, S(s));
  int* seg_tile;
  if ((err = tmp_alloc(&seg_tile, nseg, s)) || (err = tmp_alloc(&sp->seg_target, nseg, s))) return err;
  k_split_keys<<<grid_for(nseg, 256), 256, 0, S(s)>>>(ukeys, nseg, seg_tile, sp->seg_target);
  if ((err = tmp_alloc(&sp->tile_seg_ptr, n_tiles + 1, s))) return err;
  k_int_seg_ptr<<<grid_for((nseg > n_tiles + 1 ? nseg : n_tiles + 1), 256), 256, 0, S(s)>>>(seg_tile, nseg, n_tiles,
                                                                                          sp->tile_seg_ptr);
  {  // per-tile maxima of segments and contributions (the kernel stages a tile's plan in smem)
    int* mx;
    if ((err = tmp_alloc(&mx, 2, s)) || (err = tmp_alloc(&sp->tile_con_ptr, n_tiles + 1, s))) return err;
    cudaMemsetAsync(mx, 0, 2 * sizeof(int), S(s));
    k_tile_max<<<grid_for(n_tiles + 1, 256), 256, 0, S(s)>>>(sp->tile_seg_ptr, sp->seg_con_ptr, n_tiles, mx,
                                                             sp->tile_con_ptr);
    int h[2];
    cudaMemcpyAsync(h, mx, sizeof h, cudaMemcpyDeviceToHost, S(s));
    if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
    sp->max_tile_seg = h[0];
    sp->max_tile_con = h[1];
    cudaFreeAsync(mx, S(s));
    if (h[1] > 65535) return (int)cudaErrorInvalidValue;  // 16-bit relative contribution offsets
    if ((err = tmp_alloc(&sp->seg_rel, nseg > 0 ? nseg : 1, s))) return err;
    k_seg_rel<<<grid_for(nseg, 256), 256, 0, S(s)>>>(seg_tile, sp->seg_con_ptr, sp->tile_con_ptr, nseg, sp->seg_rel);
  }
  cudaFreeAsync(ukeys, S(s));
  cudaFreeAsync(counts, S(s));
  cudaFreeAsync(d_nseg, S(s));
  cudaFreeAsync(seg_tile, S(s));
  cudaFreeAsync(k2, S(s));
  // Hessian: mirrors (lower blocks written as transposes) and the touched mask
  unsigned char* touched = nullptr;
  if (row_ptr) {
    if ((err = tmp_alloc(&sp->seg_mirror, nseg, s)) || (err = tmp_alloc(&touched, n_targets, s))) return err;
    cudaMemsetAsync(touched, 0, n_targets ? n_targets : 1, S(s));
    k_seg_mirror<<<grid_for(nseg, 256), 256, 0, S(s)>>>(sp->seg_target, nseg, row_ptr, n_rows, col_idx, sp->seg_mirror,
                                                         touched);
  }
  // ownership: targets touched by one tile are written directly
  int* tcount;
  if ((err = tmp_alloc(&tcount, n_targets, s))) return err;
  cudaMemsetAsync(tcount, 0, sizeof(int) * (n_targets ? n_targets : 1), S(s));
  k_count_targets<<<grid_for(nseg, 256), 256, 0, S(s)>>>(sp->seg_target, nseg, tcount);
  int *segidx, *st2, *si2, *flag, *pos;
  if ((err = tmp_alloc(&segidx, nseg, s)) || (err = tmp_alloc(&st2, nseg, s)) || (err = tmp_alloc(&si2, nseg, s)) ||
      (err = tmp_alloc(&flag, nseg + 1, s)) || (err = tmp_alloc(&pos, nseg + 1, s)))
    return err;
  k_iota<<<grid_for(nseg, 256), 256, 0, S(s)>>>(segidx, nseg);
  tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, sp->seg_target, st2, segidx, si2, nseg, 0, bits_for(n_targets), S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceRadixSort::SortPairs(tmp, tb, sp->seg_target, st2, segidx, si2, nseg, 0, bits_for(n_targets), S(s));
  cudaFreeAsync(tmp, S(s));
  k_boundary_flags<<<grid_for(nseg, 256), 256, 0, S(s)>>>(st2, nseg, tcount, flag);
  cudaMemsetAsync(flag + nseg, 0, sizeof(int), S(s));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, nseg + 1, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, nseg + 1, S(s));
  cudaFreeAsync(tmp, S(s));
  if ((err = tmp_alloc(&sp->seg_dst, nseg, s))) return err;
  k_seg_dst<<<grid_for(nseg, 256), 256, 0, S(s)>>>(st2, si2, flag, pos, nseg, sp->seg_dst);
  long long npart = 0;
  { int v = 0; cudaMemcpyAsync(&v, pos + nseg, sizeof(int), cudaMemcpyDeviceToHost, S(s));
    if ((err = (int)cudaStreamSynchronize(S(s)))) return err; npart = v; }
  sp->n_partials = npart;
  // partial targets: boundary entries of the target-sorted list, grouped by target (tile order)
  int *btarget, *d_nb;
  if ((err = tmp_alloc(&btarget, npart, s)) || (err = tmp_alloc(&d_nb, 1, s))) return err;
  tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, st2, flag, btarget, d_nb, nseg, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceSelect::Flagged(tmp, tb, st2, flag, btarget, d_nb, nseg, S(s));
  cudaFreeAsync(tmp, S(s));
  int *pcounts, *d_npt;
  if ((err = tmp_alloc(&sp->pt_target, npart, s)) || (err = tmp_alloc(&pcounts, npart + 1, s)) ||
      (err = tmp_alloc(&d_npt, 1, s)))
    return err;
  tb = 0;
  cub::DeviceRunLengthEncode::Encode(nullptr, tb, btarget, sp->pt_target, pcounts, d_npt, npart, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceRunLengthEncode::Encode(tmp, tb, btarget, sp->pt_target, pcounts, d_npt, npart, S(s));
  cudaFreeAsync(tmp, S(s));
  int npt = 0;
  cudaMemcpyAsync(&npt, d_npt, sizeof(int), cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  sp->n_pt = npt;
  if ((err = tmp_alloc(&sp->pt_ptr, (long long)npt + 1, s))) return err;
  cudaMemsetAsync(pcounts + npt, 0, sizeof(int), S(s));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, pcounts, sp->pt_ptr, npt + 1, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceScan::ExclusiveSum(tmp, tb, pcounts, sp->pt_ptr, npt + 1, S(s));
  cudaFreeAsync(tmp, S(s));
  // targets nobody writes (e.g. the diagonal block of an isolated node): zeroed every assemble
  unsigned char* zflag;
  int *tidx, *d_nz;
  if ((err = tmp_alloc(&zflag, n_targets, s)) || (err = tmp_alloc(&tidx, n_targets, s)) ||
      (err = tmp_alloc(&sp->untouched, n_targets, s)) || (err = tmp_alloc(&d_nz, 1, s)))
    return err;
  if (touched) {
    k_not<<<grid_for(n_targets, 256), 256, 0, S(s)>>>(touched, n_targets, zflag);
    // partial targets also write their mirror in the fix-up
    if ((err = tmp_alloc(&sp->pt_mirror, npt, s))) return err;
    if (npt)
      k_seg_mirror<<<grid_for(npt, 256), 256, 0, S(s)>>>(sp->pt_target, npt, row_ptr, n_rows, col_idx, sp->pt_mirror,
                                                          touched);
  } else {
    k_is_zero<<<grid_for(n_targets, 256), 256, 0, S(s)>>>(tcount, n_targets, zflag);
  }
  k_iota<<<grid_for(n_targets, 256), 256, 0, S(s)>>>(tidx, n_targets);
  tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, tidx, zflag, sp->untouched, d_nz, n_targets, S(s));
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceSelect::Flagged(tmp, tb, tidx, zflag, sp->untouched, d_nz, n_targets, S(s));
  cudaFreeAsync(tmp, S(s));
  int nz = 0;
  cudaMemcpyAsync(&nz, d_nz, sizeof(int), cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  sp->n_untouched = nz;
  for (void* p : {(void*)tcount, (void*)segidx, (void*)st2, (void*)si2, (void*)flag, (void*)pos, (void*)btarget,
                  (void*)d_nb, (void*)pcounts, (void*)d_npt, (void*)zflag, (void*)tidx, (void*)d_nz})
    cudaFreeAsync(p, S(s));
  if (touched) cudaFreeAsync(touched, S(s));
  return (int)cudaGetLastError();
}

__global__ void k_minmax3(const double* __restrict__ a, long long items, int comps, unsigned long long* mm) {
  // mm[0..2] = ordered-int min, mm[3..5] = ordered-int max of the first three components
  // warp-reduce first: one atomic pair per warp and component (contention-free at 6M items)
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int c = 0; c < 3 && c < comps; ++c) {
    unsigned long long lo = ~0ull, hi = 0ull;
    if (i < items) {
      const long long bits = __double_as_longlong(a[i * comps + c]);
      lo = hi = bits < 0 ? ~(unsigned long long)bits : ((unsigned long long)bits | (1ull << 63));
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = l2 < lo ? l2 : lo;
      hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mm + c, lo);
      atomicMax(mm + 3 + c, hi);
    }
  }
}

double from_ordered(unsigned long long o) {
  const unsigned long long bits = (o >> 63) ? (o & ~(1ull << 63)) : ~o;
  double d;
  std::memcpy(&d, &bits, 8);
  return d;
}

}  // namespace

int tile_order(const LbDesc& d, const double* const* arrs_host, const int* conn, const int* active, long long n,
               int* perm, int* elems, void* s) {
  int err;
  if (n <= 0) return 0;
  // element centroids, their bounding box, 30-bit Morton keys
  unsigned long long* mm;
  const double** arrs_dev;
  double* cen;
  unsigned *key, *key2;
  int* ord;
  if ((err = tmp_alloc(&mm, 6, s)) || (err = tmp_alloc((char**)&arrs_dev, sizeof(double*) * d.n_lb, s)) ||
      (err = tmp_alloc(&cen, 3 * n, s)) || (err = tmp_alloc(&key, n, s)) || (err = tmp_alloc(&key2, n, s)) ||
      (err = tmp_alloc(&ord, n, s)))
    return err;
  const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
  cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, S(s));
  cudaMemcpyAsync(arrs_dev, arrs_host, sizeof(double*) * d.n_lb, cudaMemcpyHostToDevice, S(s));
  k_centroids<<<grid_for(n, 256), 256, 0, S(s)>>>(d, arrs_dev, conn, active, n, cen);
  k_minmax3<<<grid_for(n, 256), 256, 0, S(s)>>>(cen, n, 3, mm);
  unsigned long long h[6];
  cudaMemcpyAsync(h, mm, sizeof h, cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  // one scale for the three axes (the bounding cube of the largest extent): normalising each
  // axis separately stretched a thin axis (a cloth's z noise) over the full key range, so the
  // Morton order followed the noise and the tiles were scattered (config 4: 34.7 M segments /
  // 33.6 M partials per-axis, 12.6 M / 10.7 M with the cube)
  double lo[3], inv[3], ext = 0.0;
  for (int c = 0; c < 3; ++c) {
    lo[c] = from_ordered(h[c]);
    ext = fmax(ext, from_ordered(h[3 + c]) - lo[c]);
  }
  const bool per_axis = std::getenv("SYMEL_MORTON_PER_AXIS") != nullptr;
  for (int c = 0; c < 3; ++c) {
    const double e = per_axis ? from_ordered(h[3 + c]) - lo[c] : ext;
    inv[c] = e > 0 ? 1023.0 / e : 0.0;
  }
  k_morton_keys<<<grid_for(n, 256), 256, 0, S(s)>>>(cen, n, make_double3(lo[0], lo[1], lo[2]),
                                                    make_double3(inv[0], inv[1], inv[2]), key, ord);
  cudaFreeAsync(cen, S(s));
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, ord, perm, n, 0, 30, S(s));
  void* tmp;
  if ((err = tmp_alloc((char**)&tmp, tb, s))) return err;
  cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, ord, perm, n, 0, 30, S(s));  // stable: ties keep order
  cudaFreeAsync(tmp, S(s));
  k_compose<<<grid_for(n, 256), 256, 0, S(s)>>>(perm, active, n, elems);
  for (void* p : {(void*)mm, (void*)arrs_dev, (void*)key, (void*)ord, (void*)key2}) cudaFreeAsync(p, S(s));
  return (int)cudaStreamSynchronize(S(s));
}

int build_tile_plan(const TileSrc* src, int ne, long long n_blocks, long long n_rows, const int* row_ptr,
                    const int* col_idx, TilePlan* out, void* s) {
  int err;
  long long nh = 0, ng = 0, tiles = 0;
  for (int k = 0; k < ne; ++k) {
    nh += src[k].n_active * src[k].d.n_lb * src[k].d.n_lb;
    ng += src[k].n_active * src[k].d.n_lb;
    tiles = src[k].tile_base + (src[k].n_active + src[k].tpb - 1) / src[k].tpb;
  }
  out->n_tiles = tiles;
  unsigned long long *hk, *gk;
  unsigned short *hv, *gv;
  if ((err = tmp_alloc(&hk, nh, s)) || (err = tmp_alloc(&hv, nh, s)) || (err = tmp_alloc(&gk, ng, s)) ||
      (err = tmp_alloc(&gv, ng, s)))
    return err;
  unsigned long long ph = 0, pg = 0;
  for (int k = 0; k < ne; ++k) {
    if (src[k].n_active > 0) {
      k_tile_hkeys<<<grid_for(src[k].n_active, 128), 128, 0, S(s)>>>(src[k], ph, key_sentinel(tiles), hk, hv);
      k_tile_gkeys<<<grid_for(src[k].n_active, 128), 128, 0, S(s)>>>(src[k], pg, gk, gv);
    }
    ph += (unsigned long long)src[k].n_active * src[k].d.n_lb * src[k].d.n_lb;
    pg += (unsigned long long)src[k].n_active * src[k].d.n_lb;
  }
  // per-tile segment-sort flags (energies staging in shared memory)
  unsigned char* tsort = nullptr;
  bool any_sort = false;
  {
    std::vector<unsigned char> h((size_t)(tiles > 0 ? tiles : 1), 0);
    for (int k = 0; k < ne; ++k) {
      const long long nt = (src[k].n_active + src[k].tpb - 1) / src[k].tpb;
      for (long long t = 0; t < nt; ++t) h[(size_t)(src[k].tile_base + t)] = src[k].sort_segments ? 1 : 0;
      any_sort = any_sort || (src[k].sort_segments && nt > 0);
    }
    if (any_sort) {
      if ((err = tmp_alloc(&tsort, h.size(), s))) return err;
      cudaMemcpyAsync(tsort, h.data(), h.size(), cudaMemcpyHostToDevice, S(s));
      if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
    }
  }
  if ((err = build_segments(hk, hv, nh, tiles, n_blocks, row_ptr, col_idx, n_rows, tsort, &out->h, s))) return err;
  if ((err = build_segments(gk, gv, ng, tiles, n_rows, nullptr, nullptr, 0, tsort, &out->g, s))) return err;
  if (tsort) cudaFreeAsync(tsort, S(s));
  cudaFreeAsync(hk, S(s));
  cudaFreeAsync(hv, S(s));  // sorted copies live in SegPlan::con
  cudaFreeAsync(gk, S(s));
  cudaFreeAsync(gv, S(s));
  return (int)cudaStreamSynchronize(S(s));
}

void free_tile_plan(TilePlan* p) {
  for (SegPlan* sp : {&p->h, &p->g})
    for (void* q : {(void*)sp->tile_seg_ptr, (void*)sp->seg_target, (void*)sp->seg_con_ptr, (void*)sp->seg_rel, (void*)sp->con,
                    (void*)sp->seg_dst, (void*)sp->pt_ptr, (void*)sp->pt_target, (void*)sp->untouched,
                    (void*)sp->seg_mirror, (void*)sp->pt_mirror, (void*)sp->tile_con_ptr})
      if (q) cudaFree(q);
  *p = TilePlan{};
}

int tile_fixup(const TilePlan& p, const double* partials, const double* gpartials, int b, double* vals, double* grad,
               void* s, int which) {
  const int bb = b * b;
  if (which & 1) {
  if (p.h.n_pt && !fixup_dispatch(p.h, true, b, partials, vals, S(s)))
    k_fixup<<<grid_for(p.h.n_pt * bb, 256), 256, 0, S(s)>>>(p.h.pt_ptr, p.h.pt_target, p.h.pt_mirror, p.h.n_pt, bb, b,
                                                            partials, vals);
    if (p.h.n_untouched)
      k_zero_targets<<<grid_for(p.h.n_untouched * bb, 256), 256, 0, S(s)>>>(p.h.untouched, p.h.n_untouched, bb, vals);
  }
  if (which & 2) {
    if (p.g.n_pt && !fixup_dispatch(p.g, false, b, gpartials, grad, S(s)))
      k_fixup<<<grid_for(p.g.n_pt * b, 256), 256, 0, S(s)>>>(p.g.pt_ptr, p.g.pt_target, nullptr, p.g.n_pt, b, b,
                                                             gpartials, grad);
    if (p.g.n_untouched)
      k_zero_targets<<<grid_for(p.g.n_untouched * b, 256), 256, 0, S(s)>>>(p.g.untouched, p.g.n_untouched, b, grad);
  }
  return (int)cudaGetLastError();
}

__global__ void k_soa_gather(const double* __restrict__ src, int comps, const int* __restrict__ map, long long n,
                             long long stride, double* __restrict__ dst) {
  const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const long long el = map ? (long long)map[pos] : pos;
  for (int c = 0; c < comps; ++c) dst[(long long)c * stride + pos] = src[el * comps + c];
}

// tile-ordered connectivity, slot-major: dst[k * n + pos] = conn[map[pos] * arity + k]
__global__ void k_conn_soa(const int* __restrict__ conn, int arity, const int* __restrict__ map, long long n,
                           int* __restrict__ dst) {
  const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const long long el = map ? (long long)map[pos] : pos;
  for (int k = 0; k < arity; ++k) dst[(long long)k * n + pos] = conn[el * arity + k];
}

int conn_soa(const int* conn, int arity, const int* map, long long n, int* dst, void* s) {
  if (n > 0) k_conn_soa<<<grid_for(n, 256), 256, 0, S(s)>>>(conn, arity, map, n, dst);
  return (int)cudaGetLastError();
}

int soa_gather(const double* src, int comps, const int* map, long long n, long long stride, double* dst, void* s) {
  if (n > 0) k_soa_gather<<<grid_for(n, 256), 256, 0, S(s)>>>(src, comps, map, n, stride, dst);
  return (int)cudaGetLastError();
}

// only the listed component rows: dst[r * stride + pos] = src[map[pos] * comps + rows[r]]
__global__ void k_soa_gather_rows(const double* __restrict__ src, int comps, const int* __restrict__ rows, int n_rows,
                                  const int* __restrict__ map, long long n, long long stride, double* __restrict__ dst) {
  const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const long long el = map ? (long long)map[pos] : pos;
  for (int r = 0; r < n_rows; ++r) dst[(long long)r * stride + pos] = src[el * comps + __ldg(rows + r)];
}

int soa_gather_rows(const double* src, int comps, const int* rows, int n_rows, const int* map, long long n,
                    long long stride, double* dst, void* s) {
  if (n > 0 && n_rows > 0)
    k_soa_gather_rows<<<grid_for(n, 256), 256, 0, S(s)>>>(src, comps, rows, n_rows, map, n, stride, dst);
  return (int)cudaGetLastError();
}

// Component classes of a per-item array (items x comps, AoS): pass 1 accumulates per component a
// position-dependent 64-bit hash sum and the OR of the bit patterns over all items; the host
// groups components with equal sums; pass 2 verifies every grouped component against its
// representative bit for bit (a mismatch anywhere makes the component its own class).
__global__ void k_comp_hash(const unsigned long long* __restrict__ src, int comps, long long items,
                            unsigned long long* __restrict__ hsum, unsigned long long* __restrict__ hor) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;  // component (fast index: coalesced rows)
  if (c >= comps) return;
  unsigned long long sum = 0ull, orv = 0ull;
  for (long long i = blockIdx.x; i < items; i += gridDim.x) {
    const unsigned long long v = src[i * comps + c];
    unsigned long long z = v + 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    sum += z ^ (z >> 31);
    orv |= v;
  }
  atomicAdd(hsum + c, sum);
  atomicOr(hor + c, orv);
}

__global__ void k_comp_verify(const unsigned long long* __restrict__ src, int comps, long long items,
                              const int* __restrict__ rep, int* __restrict__ differs) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= comps) return;
  const int r = rep[c];
  if (r == c || r < 0) return;
  bool bad = false;
  for (long long i = blockIdx.x; i < items; i += gridDim.x) bad = bad || src[i * comps + c] != src[i * comps + r];
  if (bad) differs[c] = 1;
}

int comp_classes(const double* src, int comps, long long items, int* cls, void* s) {
  for (int c = 0; c < comps; ++c) cls[c] = c;
  if (items <= 0 || comps <= 0) return 0;
  int err;
  unsigned long long *hsum = nullptr, *hor = nullptr;
  int *rep = nullptr, *differs = nullptr;
  if ((err = tmp_alloc(&hsum, comps, s)) || (err = tmp_alloc(&hor, comps, s)) || (err = tmp_alloc(&rep, comps, s)) ||
      (err = tmp_alloc(&differs, comps, s)))
    return err;
  cudaMemsetAsync(hsum, 0, sizeof(unsigned long long) * comps, S(s));
  cudaMemsetAsync(hor, 0, sizeof(unsigned long long) * comps, S(s));
  cudaMemsetAsync(differs, 0, sizeof(int) * comps, S(s));
  const int tx = comps >= 128 ? 128 : (comps >= 64 ? 64 : 32);
  const dim3 grid((unsigned)std::min<long long>(items, 148 * 16), (unsigned)((comps + tx - 1) / tx));
  k_comp_hash<<<grid, tx, 0, S(s)>>>((const unsigned long long*)src, comps, items, hsum, hor);
  std::vector<unsigned long long> hs(comps), ho(comps);
  cudaMemcpyAsync(hs.data(), hsum, sizeof(unsigned long long) * comps, cudaMemcpyDeviceToHost, S(s));
  cudaMemcpyAsync(ho.data(), hor, sizeof(unsigned long long) * comps, cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  std::vector<int> r(comps);
  for (int c = 0; c < comps; ++c) {
    r[c] = c;
    if (ho[c] == 0ull) { r[c] = -1; continue; }  // every item holds +0.0
    for (int q = 0; q < c; ++q)
      if (r[q] == q && hs[q] == hs[c]) { r[c] = q; break; }
  }
  cudaMemcpyAsync(rep, r.data(), sizeof(int) * comps, cudaMemcpyHostToDevice, S(s));
  k_comp_verify<<<grid, tx, 0, S(s)>>>((const unsigned long long*)src, comps, items, rep, differs);
  std::vector<int> df(comps);
  cudaMemcpyAsync(df.data(), differs, sizeof(int) * comps, cudaMemcpyDeviceToHost, S(s));
  if ((err = (int)cudaStreamSynchronize(S(s)))) return err;
  for (int c = 0; c < comps; ++c) cls[c] = df[c] ? c : r[c];
  for (void* q : {(void*)hsum, (void*)hor, (void*)rep, (void*)differs}) cudaFreeAsync(q, S(s));
  return (int)cudaGetLastError();
}

int tile_energy(const double* tileE, long long first, long long n, double* partial, double* out, void* s) {
  return energy_tree(tileE + first, 1, n, partial, out, s);
}

// =================================================================== SPD projection (K2)
//
// Per element: H -> V max(L, 0) V^T for the symmetric n x n element Hessian (new component;
// the reference regularises with H + tau I instead, optimizer.hpp:196-221). Eigensystem by
// Householder tridiagonalisation + implicit QL with Wilkinson-style shifts (the classic
// tred2 / tql2 pair, Wilkinson & Reinsch; restated here), one thread per element.

namespace {

template <int N>
__device__ void sym_eig(double (&V)[N][N], double (&d)[N], double (&e)[N]) {
  // tred2: V holds the matrix on entry, the orthogonal transformation on exit
  for (int j = 0; j < N; ++j) d[j] = V[N - 1][j];
  for (int i = N - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (int k = 0; k < i; ++k) scale += fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (int j = 0; j < i; ++j) {
        d[j] = V[i - 1][j];
        V[i][j] = 0.0;
        V[j][i] = 0.0;
      }
    } else {
      for (int k = 0; k < i; ++k) {
        d[k] /= scale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h -= f * g;
      d[i - 1] = f - g;
      for (int j = 0; j < i; ++j) e[j] = 0.0;
      for (int j = 0; j < i; ++j) {
        f = d[j];
        V[j][i] = f;
        g = e[j] + V[j][j] * f;
        for (int k = j + 1; k <= i - 1; ++k) {
          g += V[k][j] * d[k];
          e[k] += V[k][j] * f;
        }
        e[j] = g;
      }
      f = 0.0;
      for (int j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      const double hh = f / (h + h);
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        for (int k = j; k <= i - 1; ++k) V[k][j] -= (f * e[k] + g * d[k]);
        d[j] = V[i - 1][j];
        V[i][j] = 0.0;
      }
    }
    d[i] = h;
  }
  for (int i = 0; i < N - 1; ++i) {
    V[N - 1][i] = V[i][i];
    V[i][i] = 1.0;
    const double h = d[i + 1];
    if (h != 0.0) {
      for (int k = 0; k <= i; ++k) d[k] = V[k][i + 1] / h;
      for (int j = 0; j <= i; ++j) {
        double g = 0.0;
        for (int k = 0; k <= i; ++k) g += V[k][i + 1] * V[k][j];
        for (int k = 0; k <= i; ++k) V[k][j] -= g * d[k];
      }
    }
    for (int k = 0; k <= i; ++k) V[k][i + 1] = 0.0;
  }
  for (int j = 0; j < N; ++j) {
    d[j] = V[N - 1][j];
    V[N - 1][j] = 0.0;
  }
  V[N - 1][N - 1] = 1.0;
  e[0] = 0.0;
  // tql2: implicit QL on the tridiagonal (d, e), rotations accumulated into V
  for (int i = 1; i < N; ++i) e[i - 1] = e[i];
  e[N - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < N; ++l) {
    tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
    int m = l;
    while (m < N - 1 && fabs(e[m]) > eps * tst1) ++m;
    if (m > l) {
      for (int iter = 0; iter < 60; ++iter) {
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = hypot(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int i = l + 2; i < N; ++i) d[i] -= h;
        f += h;
        p = d[m];
        double c = 1.0, c2 = 1.0, c3 = 1.0, s = 0.0, s2 = 0.0;
        const double el1 = e[l + 1];
        for (int i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          for (int k = 0; k < N; ++k) {
            h = V[k][i + 1];
            V[k][i + 1] = s * V[k][i] + c * h;
            V[k][i] = c * V[k][i] - s * h;
          }
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
        if (!(fabs(e[l]) > eps * tst1)) break;
      }
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
}

// In place on the full n x n Hessian block of each element's contrib row (symmetric on exit).
template <int N>
__global__ void __launch_bounds__(64) k_spd_contrib(double* __restrict__ contrib, long long stride, long long off,
                                                    long long n) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double* H = contrib + t * stride + off;
  double V[N][N], d[N], e[N];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) V[i][j] = 0.5 * (H[i * N + j] + H[j * N + i]);
  sym_eig<N>(V, d, e);
  for (int k = 0; k < N; ++k) d[k] = d[k] > 0.0 ? d[k] : 0.0;
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j) {
      double acc = 0.0;
      for (int k = 0; k < N; ++k) acc += V[i][k] * d[k] * V[j][k];
      H[i * N + j] = acc;
      H[j * N + i] = acc;
    }
}

// Per-element atomic scatter from contrib rows (K3' for paths that stage elements in global).
__global__ void k_scatter_atomic(const double* __restrict__ contrib, long long stride, int nd, int nl, int b,
                                 const signed char* __restrict__ dof_of_dummy, const int* __restrict__ slots,
                                 const int* __restrict__ conn, const int* __restrict__ active, LbDesc d, long long n,
                                 long long set_off_unused, double* __restrict__ vals, double* __restrict__ grad) {
  (void)dof_of_dummy;
  (void)set_off_unused;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double* row = contrib + t * stride;
  const long long e = active ? active[t] : t;
  const int* tup = conn + e * d.arity;
  // node-major binding: dof (li, r) = li * b + r
  for (int li = 0; li < nl; ++li) {
    const long long g0 = d.off[li] + (long long)tup[d.slot[li]] * d.comps[li];
    for (int r = 0; r < b; ++r) atomicAdd(grad + g0 + r, row[1 + li * b + r]);
    for (int lj = 0; lj < nl; ++lj) {
      double* blk = vals + (long long)slots[(t * nl + li) * nl + lj] * b * b;
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) atomicAdd(blk + r * b + c, row[1 + nd + (li * b + r) * nd + lj * b + c]);
    }
  }
}

}  // namespace

int spd_project_contrib(double* contrib, long long stride, int n_dofs, long long n_elem, void* s) {
  if (n_elem <= 0) return 0;
  const long long off = 1 + n_dofs;
  switch (n_dofs) {
    case 3: k_spd_contrib<3><<<grid_for(n_elem, 64), 64, 0, S(s)>>>(contrib, stride, off, n_elem); break;
    case 6: k_spd_contrib<6><<<grid_for(n_elem, 64), 64, 0, S(s)>>>(contrib, stride, off, n_elem); break;
    case 9: k_spd_contrib<9><<<grid_for(n_elem, 64), 64, 0, S(s)>>>(contrib, stride, off, n_elem); break;
    case 12: k_spd_contrib<12><<<grid_for(n_elem, 64), 64, 0, S(s)>>>(contrib, stride, off, n_elem); break;
    default: return (int)cudaErrorNotSupported;
  }
  return (int)cudaGetLastError();
}

int scatter_atomic_contrib(const double* contrib, long long stride, int n_dofs, const LbDesc& d, const int* slots,
                           const int* conn, const int* active, long long n, double* vals, double* grad, void* s) {
  if (n <= 0) return 0;
  k_scatter_atomic<<<grid_for(n, 128), 128, 0, S(s)>>>(contrib, stride, n_dofs, d.n_lb, d.b, nullptr, slots, conn,
                                                       active, d, n, 0, vals, grad);
  return (int)cudaGetLastError();
}

}  // namespace symel_cuda::dev
