// Microbenchmark: do DMMA (mma.sync f64) and DFMA share the FP64 datapath on sm_100a?
// Runs DMMA-only, DFMA-only and an interleaved mix; if the mix reaches ~the sum of the
// two, they are separate pipes.  Also: the fp64 rcp.approx (MUFU) + Newton throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void mix(double* out, int iters, double a, double b) {
  double c0[NM > 0 ? NM : 1], c1[NM > 0 ? NM : 1], f[NF > 0 ? NF : 1];
  double x = threadIdx.x * 1e-3, y = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int c = 0; c < NM; ++c) c0[c] = c1[c] = 0;
#pragma unroll
  for (int c = 0; c < NF; ++c) f[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NM; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(x), "d"(y));
#pragma unroll
    for (int c = 0; c < NF; ++c) f[c] = fma(f[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NM; ++c) s += c0[c] + c1[c];
#pragma unroll
  for (int c = 0; c < NF; ++c) s += f[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void rcp_loop(double* out, int iters) {
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = 1.5 + threadIdx.x * 1e-6 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double y;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v[c]));
      v[c] = y + 1.0;
    }
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += v[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NM, int NF>
void run(const char* name, int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int tpb = 256, bps = 2, iters = 20000;
  dim3 g(sms * bps);
  mix<NM, NF><<<g, tpb>>>(out, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  mix<NM, NF><<<g, tpb>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double thr = (double)g.x * tpb;
  const double fm = 2.0 * 256 / 32 * NM * (double)iters * thr;  // 8x8x4 = 256 FMA per warp-mma
  const double ff = 2.0 * NF * (double)iters * thr;
  printf("%-14s DMMA %.2f + DFMA %.2f = %.2f TFLOP/s  (%.3f ms)\n", name, fm / ms / 1e9, ff / ms / 1e9,
         (fm + ff) / ms / 1e9, ms);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run<4, 0>("dmma only", p.multiProcessorCount, out);
  run<0, 8>("dfma only", p.multiProcessorCount, out);
  run<2, 8>("mix 2:8", p.multiProcessorCount, out);
  run<4, 8>("mix 4:8", p.multiProcessorCount, out);
  run<4, 16>("mix 4:16", p.multiProcessorCount, out);
  run<1, 8>("mix 1:8", p.multiProcessorCount, out);
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dim3 g(p.multiProcessorCount * 2);
    rcp_loop<<<g, 256>>>(out, 100);
    cudaEventRecord(e0);
    rcp_loop<<<g, 256>>>(out, 20000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rcp.approx.f64: %.1f G/s (+1 DADD each)\n", 8.0 * 20000 * g.x * 256 / ms / 1e6);
  }
  return 0;
}
