// Probe: FP64 (DFMA / DMUL / DADD), MUFU.RSQ64H and MUFU.RCP64H dependent-issue latency and the
// per-SM DFMA throughput vs resident warps on this GPU (B200: which ILP the tile kernels need).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64p scripts/fp64_latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(double* out, long long* cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-9, b = 0.999999999, c = 1e-12;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x = fma(x, b, c);
      if (OP == 1) x = x * b;
      if (OP == 2) x = x + c;
      if (OP == 3) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
      if (OP == 4) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int ILP>
__global__ void thr(double* out, int iters) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = 1.0 + k + threadIdx.x * 1e-9;
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], b, c);
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, sizeof(double) * 148 * 2048 * 4);
  cudaMalloc(&cyc, sizeof(long long) * 1024);
  const int iters = 4000;
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H", "MUFU.RCP64H"};
  for (int op = 0; op < 5; ++op) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) lat<0><<<1, 32>>>(out, cyc, iters);
      if (op == 1) lat<1><<<1, 32>>>(out, cyc, iters);
      if (op == 2) lat<2><<<1, 32>>>(out, cyc, iters);
      if (op == 3) lat<3><<<1, 32>>>(out, cyc, iters);
      if (op == 4) lat<4><<<1, 32>>>(out, cyc, iters);
      cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    }
    printf("%-12s dependent latency %.2f cycles\n", names[op], (double)h / (iters * 8.0));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int warps : {4, 8, 12, 16, 32}) {
    for (int ilp : {1, 2, 4, 8}) {
      const int it = 20000 / ilp;
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (ilp == 1) thr<1><<<148, 32 * warps>>>(out, it);
        if (ilp == 2) thr<2><<<148, 32 * warps>>>(out, it);
        if (ilp == 4) thr<4><<<148, 32 * warps>>>(out, it);
        if (ilp == 8) thr<8><<<148, 32 * warps>>>(out, it);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double flops = 2.0 * 148 * 32 * warps * (double)it * ilp;
      printf("warps/SM %2d ILP %d: %.2f TFLOP/s\n", warps, ilp, flops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
