// Microbenchmark: L1-resident contiguous warp loads, 8 vs 16 bytes per lane (same total bytes).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l1_width l1_width.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W>  // W = doubles per lane per load
__global__ void __launch_bounds__(256, 4) k(const double* __restrict__ x, double* out, int iters, int span) {
  const int t = threadIdx.x;
  double acc = 0.0;
  // each CTA walks a private 32 KB region (L1-resident after the first touch)
  const double* base = x + (size_t)blockIdx.x * span;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int q = 0; q < span / (256 * W); ++q) {
      if constexpr (W == 1) {
        acc += __ldg(base + q * 256 + t);
      } else {
        const double2 v = __ldg(reinterpret_cast<const double2*>(base) + q * 256 + t);
        acc += v.x + v.y;
      }
    }
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  const int span = 4096;  // doubles per CTA = 32 KB
  const int grid = 148 * 4, iters = 2000;
  double *x, *out;
  cudaMalloc(&x, sizeof(double) * (size_t)span * grid);
  cudaMemset(x, 0, sizeof(double) * (size_t)span * grid);
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms1, ms2;
    cudaEventRecord(e0);
    k<1><<<grid, 256>>>(x, out, iters, span);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0);
    k<2><<<grid, 256>>>(x, out, iters, span);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms2, e0, e1);
    const double bytes = 8.0 * span * (double)grid * iters;
    printf("8 B/lane: %.3f ms  %.1f B/clk/SM-equivalent at 1.9 GHz   16 B/lane: %.3f ms  %.1f\n", ms1,
           bytes / (ms1 * 1e-3) / 148 / 1.9e9, ms2, bytes / (ms2 * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
