// Probe: does launching a compute-bound, 2-CTA/SM kernel (110 KB smem, 128 threads -- the
// shape of the fused SPD tile kernel) as thread-block clusters cost SM residency?
// Times the same FP64 work with cluster sizes 1, 2, 4, 8 (and reports max active clusters).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128, 2) work(double* out, int iters) {
  extern __shared__ double sm[];
  double a = threadIdx.x * 1e-3 + blockIdx.x, b = 1.0000001, c = 0.9999999, d = 1.0;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, b, c); x1 = fma(x1, c, b); x2 = fma(x2, b, d); x3 = fma(x3, d, c);
  }
  sm[threadIdx.x] = x0 + x1 + x2 + x3;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
}

int main() {
  const int grid = 46880, smem = 110 * 1024, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * grid);
  cudaFuncSetAttribute(work, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(work, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int cl : {1, 2, 4, 8, 1}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int max_clusters = 0;
    cudaOccupancyMaxActiveClusters(&max_clusters, (void*)work, &cfg);
    cudaLaunchKernelEx(&cfg, work, out, iters);  // warm
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, work, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster %d: %.3f ms per launch, max active clusters %d (= %d CTAs), err %s\n", cl, ms / 3, max_clusters,
           max_clusters * cl, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
