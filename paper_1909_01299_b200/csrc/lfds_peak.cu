// In-run FP64 tensor-pipe peak (lfds_fp64_peak, include/lfds.h): the roofline denominator of
// the DMMA-bound kernels, measured in the same process and clock state as the solve.
#include <cuda_runtime.h>

#include "../../include/lfds.h"

namespace {

// 8 independent m8n8k4 accumulator chains per warp: enough in flight to saturate the pipe
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c0[8], c1[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) c0[c] = c1[c] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // never true: keeps the loop alive
}

}  // namespace

extern "C" int lfds_fp64_peak(void* stream, double* tflops) {
  if (!tflops) return LFDS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LFDS_ECUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return LFDS_ECUDA;
  double* out = nullptr;
  if (cudaMallocAsync(&out, 256 * sizeof(double), st) != cudaSuccess) return LFDS_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  const dim3 grid(2 * sms);
  k_dmma_peak<<<grid, 256, 0, st>>>(out, 200);  // warm-up
  cudaEventRecord(e0, st);
  k_dmma_peak<<<grid, 256, 0, st>>>(out, iters);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  if (e != cudaSuccess || ms <= 0) return LFDS_ECUDA;
  // per warp and iteration: 8 MMAs of 8 x 8 x 4 FMAs
  const double fma = (double)iters * 8 * 256.0 * grid.x / 32 * 8 * 8 * 4;
  *tflops = 2.0 * fma / (ms * 1e-3) / 1e12;
  return LFDS_OK;
}
