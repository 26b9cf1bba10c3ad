// K9 microbenchmark: FP64 peaks on sm_100a (DFMA pipe vs DMMA tensor pipe) and HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int CH>
__global__ void dmma_m8n8k4_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c0[CH], c1[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { c0[c] = 0; c1[c] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int CH>
__global__ void dmma_m16n8k16_loop(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - threadIdx.x * 1e-4 * j;
  double c[CH][4];
#pragma unroll
  for (int q = 0; q < CH; ++q) for (int j = 0; j < 4; ++j) c[q][j] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < CH; ++q)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int q = 0; q < CH; ++q) for (int j = 0; j < 4; ++j) s += c[q][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void read_kernel(const double2* __restrict__ a, double* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s = 0; for (; i < n; i += st) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int tpb : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
    if (tpb * bps > 2048) continue;
    int iters = 20000; dim3 g(sms * bps);
    dfma_loop<8><<<g, tpb>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_loop<8><<<g, tpb>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)g.x * tpb;
    printf("DFMA   tpb %4d bps %d : %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int iters = 20000; dim3 g(sms * bps);
    dmma_m8n8k4_loop<4><<<g, tpb>>>(out, 100);
    cudaEventRecord(e0); dmma_m8n8k4_loop<4><<<g, tpb>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 4 * iters * (double)g.x * (tpb / 32);
    printf("DMMA m8n8k4  tpb %4d bps %d : %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) for (int bps : {1, 2}) {
    int iters = 5000; dim3 g(sms * bps);
    dmma_m16n8k16_loop<2><<<g, tpb>>>(out, 100);
    cudaEventRecord(e0); dmma_m16n8k16_loop<2><<<g, tpb>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 16 * 2 * iters * (double)g.x * (tpb / 32);
    printf("DMMA m16n8k16 tpb %4d bps %d : %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
  }
  size_t n = (size_t)1 << 28; // 4 GiB of double2
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy double2: %.1f GB/s (r+w)\n", 2.0 * n * 16 / ms / 1e6);
    cudaEventRecord(e0); read_kernel<<<sms * 8, 512>>>(a, out, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read double2: %.1f GB/s\n", 1.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
