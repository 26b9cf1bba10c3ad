// Resonance margins of the z-systems (reading R13; SPEC S:273, S:291, S:303 via SURVEY §8(b)):
// the block z-systems T_lm = A' + (lambda_l + mu_m) E of steps 2 and 6
// and the global ones of step 5 are singular exactly when
// lambda_l + mu_m + theta_t = 0 for a z-pencil eigenvalue theta_t (A' z = theta E z).  Setup
// takes min |lambda_l + mu_m + theta_t| over every (l, m, t) of every block and of the global
// bases on the device (about N_x N_y N_z complex sums per family: milliseconds) and reports the
// minimum with its harmonic, never regularising (lfds_setup_grid returns LFDS_ERESONANCE).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lfds_internal.h"

namespace lfds {

namespace {

// key = (float bits of |lambda_l + mu_m + theta_t|) << 32 | flat index: non-negative floats
// order like their bit patterns, so one 64-bit atomicMin keeps the minimum and its argmin
__global__ void __launch_bounds__(256) k_margin(const double2* __restrict__ ev, const MarginSet* __restrict__ sets,
                                                const double2* __restrict__ theta, int nz,
                                                unsigned long long* __restrict__ out) {
  const MarginSet S = sets[blockIdx.y];
  const uint32_t total = (uint32_t)S.nx * (uint32_t)S.ny * (uint32_t)nz;
  unsigned long long best = ~0ull;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t l = i % (uint32_t)S.nx, r = i / (uint32_t)S.nx;
    const uint32_t m = r % (uint32_t)S.ny, t = r / (uint32_t)S.ny;
    const double2 a = ev[S.lx + l], b = ev[S.ly + m], c = theta[t];
    const double re = a.x + b.x + c.x, im = a.y + b.y + c.y;
    const float mag = (float)sqrt(re * re + im * im);
    const unsigned long long key = ((unsigned long long)__float_as_uint(mag) << 32) | i;
    best = key < best ? key : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v < best ? v : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(out + blockIdx.y, best);
}

}  // namespace

cudaError_t launch_margins(const double2* d_ev, const MarginSet* d_sets, int nsets, const double2* d_theta, int nz,
                           unsigned long long* d_out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_out, 0xff, sizeof(unsigned long long) * nsets, st);
  if (e != cudaSuccess) return e;
  for (int s0 = 0; s0 < nsets; s0 += 65535) {
    const int ns = nsets - s0 < 65535 ? nsets - s0 : 65535;
    k_margin<<<dim3(nsets == 1 ? 592 : 32, ns), 256, 0, st>>>(d_ev, d_sets + s0, d_theta, nz, d_out + s0);
  }
  return cudaGetLastError();
}

}  // namespace lfds
