// Two-sided few-row projections of a mode plane, read once (FP64 CUDA cores):
//
//   G[e][p][m] = sum_l Wr[e][l] X[p][m][l]      (e < E1)
//   H[e][p][l] = sum_m Wc[e][m] X[p][m][l]      (e < E2)
//
//  * step 3: X = a block's v~, Wr / Wc = the first and last rows of
//    W_x / W_y, so G and H are the partial inverse transforms that give v on the rows next
//    to every block face (E1 = E2 = 2);
//  * step 5: X = the global correction w^ in mode space, Wr = W_x[I_a, :],
//    Wc = W_y[I_b, :], so G = P1 and H = P2 are w^ projected onto the interface planes
//    (E = |I_x|, |I_y|).
// One CTA per plane p: thread t owns the columns l = t + j*blockDim (j < LPT) and streams
// the rows m, RB at a time (loads of the next batch in flight while the current one is
// used).  H accumulates in registers over all m (no reduction).  G needs a sum over l:
// each warp does a reduce-scatter through shuffles (2E doubles over 32 lanes in 2E-1+...
// = ~2E shuffles instead of 10E), the NW per-warp partials go through shared memory and
// are summed in a fixed order (deterministic).  HBM-bound: 16 B per element read.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lfds_internal.h"

namespace lfds {
namespace {

constexpr int RB = 4;  // rows per batch

template <int N>  // N doubles (power of two, 2..32) reduced over the warp; lane ends with one
__device__ __forceinline__ double reduce_scatter(double (&v)[N], int& idx) {
  const int lane = threadIdx.x & 31;
  idx = 0;
  int cnt = N;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int off = 16 >> s;
    if (cnt > 1) {
      const int h = cnt / 2;
      const bool upper = lane & off;
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        if (i < h) {
          const double send = upper ? v[i] : v[h + i];
          const double keep = upper ? v[h + i] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (upper) idx += h;
      cnt = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

template <int E, int LPT>
__global__ void __launch_bounds__(512) k_proj(const PDesc* __restrict__ descs, Bufs bufs) {
  constexpr int N = 2 * E;
  extern __shared__ double red[];  // [2][RB][NW][N]
  const PDesc& D = descs[blockIdx.y];
  const int p = blockIdx.x;
  if (p >= D.nplanes) return;
  const int NW = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx = D.nx, ny = D.ny, E1 = D.E1, E2 = D.E2;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* X = reinterpret_cast<const double2*>(bufs.p[D.x_buf]) + D.x_off + (int64_t)p * D.ps;
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  int lj[LPT];
  bool ok[LPT];
  double2 wr[LPT][E], h[LPT][E];
#pragma unroll
  for (int j = 0; j < LPT; ++j) {
    lj[j] = threadIdx.x + j * blockDim.x;
    ok[j] = lj[j] < nx;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      wr[j][e] = (ok[j] && e < E1) ? __ldg(TAB + D.wr + (int64_t)e * D.wr_es + lj[j]) : make_double2(0, 0);
      h[j][e] = make_double2(0, 0);
    }
  }
  double2 xc[RB][LPT], xn[RB][LPT];  // current batch, next batch (in flight)
  auto load = [&](double2 (&xb)[RB][LPT], int m0) {
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int j = 0; j < LPT; ++j)
        xb[r][j] = (ok[j] && m0 + r < ny) ? __ldg(X + (int64_t)(m0 + r) * nx + lj[j]) : make_double2(0, 0);
  };
  const int nb = (ny + RB - 1) / RB;
  load(xn, 0);
  for (int b = 0; b < nb; ++b) {
    const int m0 = b * RB, cur = b & 1;
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int j = 0; j < LPT; ++j) xc[r][j] = xn[r][j];
    if (b + 1 < nb) load(xn, m0 + RB);
    double* rb = red + (size_t)cur * RB * NW * N;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int m = m0 + r;
      if (m >= ny) break;  // uniform over the CTA
      // H: column accumulation
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e < E2) {
          const double2 w = __ldg(TAB + D.wc + (int64_t)e * D.wc_es + m);
#pragma unroll
          for (int j = 0; j < LPT; ++j) {
            const double2 x = xc[r][j];
            h[j][e].x = fma(w.x, x.x, fma(-w.y, x.y, h[j][e].x));
            h[j][e].y = fma(w.x, x.y, fma(w.y, x.x, h[j][e].y));
          }
        }
      }
      // G: row reduction
      double g[N];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        double gx = 0, gy = 0;
#pragma unroll
        for (int j = 0; j < LPT; ++j) {
          const double2 x = xc[r][j];
          gx = fma(wr[j][e].x, x.x, fma(-wr[j][e].y, x.y, gx));
          gy = fma(wr[j][e].x, x.y, fma(wr[j][e].y, x.x, gy));
        }
        g[2 * e] = gx;
        g[2 * e + 1] = gy;
      }
      int idx;
      const double s = reduce_scatter<N>(g, idx);
      // lanes holding a unique index: the lowest lane of each group of 32/N
      if ((lane & (32 / N - 1)) == 0 || N >= 32) rb[(r * NW + warp) * N + idx] = s;
    }
    __syncthreads();
    // fixed-order sum over warps; thread -> (row, idx)
    for (int t = threadIdx.x; t < RB * N; t += blockDim.x) {
      const int r = t / N, idx = t - r * N, e = idx >> 1, m = m0 + r;
      if (m < ny && e < E1) {
        double acc = 0;
        for (int w = 0; w < NW; ++w) acc += rb[(r * NW + w) * N + idx];
        reinterpret_cast<double*>(IF + D.g_off + (int64_t)e * D.g_es + (int64_t)p * D.g_ps + m)[idx & 1] = acc;
      }
    }
    // the next batch writes the other half of red; the barrier of that batch orders reuse
  }
#pragma unroll
  for (int j = 0; j < LPT; ++j)
    if (ok[j])
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < E2) IF[D.h_off + (int64_t)e * D.h_es + (int64_t)p * D.h_ps + lj[j]] = h[j][e];
}

template <int E, int LPT>
cudaError_t launch_e(const PDesc* d, int ndesc, int maxplanes, int threads, cudaStream_t st, const Bufs& bufs) {
  const size_t sm = (size_t)2 * RB * (threads / 32) * 2 * E * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_proj<E, LPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_proj<E, LPT><<<dim3((unsigned)maxplanes, (unsigned)ndesc), threads, sm, st>>>(d, bufs);
  return cudaGetLastError();
}

template <int LPT>
cudaError_t launch_l(int E, const PDesc* d, int ndesc, int maxplanes, int threads, cudaStream_t st, const Bufs& bufs) {
  if (E <= 1) return launch_e<1, LPT>(d, ndesc, maxplanes, threads, st, bufs);
  if (E <= 2) return launch_e<2, LPT>(d, ndesc, maxplanes, threads, st, bufs);
  if (E <= 4) return launch_e<4, LPT>(d, ndesc, maxplanes, threads, st, bufs);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_proj(const PDesc* d_descs, int ndesc, int max_nx, int maxE, int maxplanes, cudaStream_t st,
                        const Bufs& bufs) {
  if (ndesc <= 0 || maxplanes <= 0) return cudaSuccess;
  if (ndesc > 65535 || max_nx > 1024) return cudaErrorInvalidValue;
  int threads = ((max_nx + 31) / 32) * 32;
  if (threads <= 512) return launch_l<1>(maxE, d_descs, ndesc, maxplanes, threads, st, bufs);
  threads = ((max_nx + 63) / 64) * 32;
  return launch_l<2>(maxE, d_descs, ndesc, maxplanes, threads, st, bufs);
}

}  // namespace lfds
