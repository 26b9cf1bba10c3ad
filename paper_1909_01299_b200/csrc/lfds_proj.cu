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

__device__ __forceinline__ void cp16p(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}

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

// Row-per-warp variant for narrow planes (block planes, nx <= 32*LPW): warp w streams rows
// m = w, w + NW, ... and each lane holds LPW columns, so a row sum of G is complete inside
// the warp (reduce-scatter) and the CTA needs no barrier in its row loop; H (column sums)
// accumulates per warp and is combined once per plane through shared memory, in warp order.
// Rows arrive through a per-warp cp.async ring PNST rows deep (each lane copies and later reads
// only its own columns, so a per-thread wait_group orders them; no warp or CTA barrier): PNST-1
// rows per warp in flight without holding them in registers.
constexpr int PNST = 4;
template <int E, int LPW>
__global__ void __launch_bounds__(128, 4) k_proj_rows(const PDesc* __restrict__ descs, Bufs bufs) {
  constexpr int N = 2 * E, NW = 4, RW = 32 * LPW;
  extern __shared__ __align__(16) double2 psm[];  // ring[NW][PNST][RW], then hs[NW][E][RW]
  const PDesc& D = descs[blockIdx.y];
  const int p = blockIdx.x;
  if (p >= D.nplanes) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx = D.nx, ny = D.ny, E1 = D.E1, E2 = D.E2;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* X = reinterpret_cast<const double2*>(bufs.p[D.x_buf]) + D.x_off + (int64_t)p * D.ps;
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  double2* ring = psm + warp * PNST * RW;
  double2 (*hs)[E][RW] = reinterpret_cast<double2 (*)[E][RW]>(psm + NW * PNST * RW);
  double2* wcs = psm + NW * PNST * RW + NW * E * RW;  // Wc[e][m], staged once per plane
  const bool wsm = ny <= RW;  // Wc fits its staging area (else read through L1 per row)
  if (wsm)
    for (int c = threadIdx.x; c < E * ny; c += blockDim.x) {
      const int e = c / ny, m = c - e * ny;
      cp16p(wcs + c, TAB + D.wc + (int64_t)e * D.wc_es + m, e < E2);
    }
  double2 wr[LPW][E], h[LPW][E];
#pragma unroll
  for (int j = 0; j < LPW; ++j) {
    const int l = lane + 32 * j;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      wr[j][e] = (l < nx && e < E1) ? __ldg(TAB + D.wr + (int64_t)e * D.wr_es + l) : make_double2(0, 0);
      h[j][e] = make_double2(0, 0);
    }
  }
  // row i of this warp is m = warp + NW*i, in slot i % PNST
  const int nrow = ny > warp ? (ny - warp + NW - 1) / NW : 0;
  auto issue = [&](int i) {
    if (i < nrow) {
      const int m = warp + NW * i;
      double2* d = ring + (i % PNST) * RW;
#pragma unroll
      for (int j = 0; j < LPW; ++j) {
        const int l = lane + 32 * j;
        const bool ok = l < nx;
        cp16p(d + l, ok ? X + (int64_t)m * nx + l : X, ok);  // zero-fill past nx
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int q = 0; q < PNST - 1; ++q) issue(q);
  asm volatile("cp.async.wait_group %0;\n" ::"n"(PNST - 2) : "memory");  // Wc rows (in the first group)
  __syncthreads();
  for (int i = 0; i < nrow; ++i) {
    const int m = warp + NW * i;
    issue(i + PNST - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PNST - 1) : "memory");
    double2 xc[LPW];
    const double2* s = ring + (i % PNST) * RW;
#pragma unroll
    for (int j = 0; j < LPW; ++j) xc[j] = s[lane + 32 * j];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e < E2) {
        const double2 w = wsm ? wcs[e * ny + m] : __ldg(TAB + D.wc + (int64_t)e * D.wc_es + m);
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
          h[j][e].x = fma(w.x, xc[j].x, fma(-w.y, xc[j].y, h[j][e].x));
          h[j][e].y = fma(w.x, xc[j].y, fma(w.y, xc[j].x, h[j][e].y));
        }
      }
    }
    double g[N];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      double gx = 0, gy = 0;
#pragma unroll
      for (int j = 0; j < LPW; ++j) {
        gx = fma(wr[j][e].x, xc[j].x, fma(-wr[j][e].y, xc[j].y, gx));
        gy = fma(wr[j][e].x, xc[j].y, fma(wr[j][e].y, xc[j].x, gy));
      }
      g[2 * e] = gx;
      g[2 * e + 1] = gy;
    }
    int idx;
    const double sum = reduce_scatter<N>(g, idx);
    if (((lane & (32 / N - 1)) == 0 || N >= 32) && (idx >> 1) < E1)
      reinterpret_cast<double*>(IF + D.g_off + (int64_t)(idx >> 1) * D.g_es + (int64_t)p * D.g_ps + m)[idx & 1] = sum;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < LPW; ++j)
#pragma unroll
    for (int e = 0; e < E; ++e) hs[warp][e][lane + 32 * j] = h[j][e];
  __syncthreads();
  for (int t = threadIdx.x; t < E * RW; t += blockDim.x) {
    const int e = t / RW, l = t % RW;
    if (e < E2 && l < nx) {
      double2 acc = hs[0][e][l];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        acc.x += hs[w][e][l].x;
        acc.y += hs[w][e][l].y;
      }
      IF[D.h_off + (int64_t)e * D.h_es + (int64_t)p * D.h_ps + l] = acc;
    }
  }
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
  if (maxE <= 2 && max_nx > 32 && max_nx <= 160) {  // wide block planes: row-per-warp variant
    const dim3 grid((unsigned)maxplanes, (unsigned)ndesc);
#define PR(LPW)                                                                                   \
  {                                                                                               \
    const int sm = ((4 * PNST + 4 * 2) * 32 * LPW + 2 * 32 * LPW) * (int)sizeof(double2);        \
    cudaError_t e = cudaFuncSetAttribute(k_proj_rows<2, LPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
    if (e != cudaSuccess) return e;                                                               \
    k_proj_rows<2, LPW><<<grid, 128, sm, st>>>(d_descs, bufs);                                    \
    return cudaGetLastError();                                                                    \
  }
    if (max_nx <= 64) PR(2)
    if (max_nx <= 128) PR(4)
    PR(5)
#undef PR
  }
  int threads = ((max_nx + 31) / 32) * 32;
  if (threads <= 512) return launch_l<1>(maxE, d_descs, ndesc, maxplanes, threads, st, bufs);
  threads = ((max_nx + 63) / 64) * 32;
  return launch_l<2>(maxE, d_descs, ndesc, maxplanes, threads, st, bufs);
}


// ============================================================================================
// Step-5 projections on the DMMA pipe (one read of the global correction w^):
//   P1[a][p][m] = sum_l W_x[I_a][l] w^[p][m][l],   P2[b][p][l] = sum_m W_y[I_b][m] w^[p][m][l]
// (w on the interface planes needs only these rows of the inverse transform).
// CTA = one l-chunk of up to 256 columns of one plane p, all rows m in tiles of 8 staged by
// cp.async (double-buffered).  Per tile and warp (32 columns):
//   P2 (K = m):  C[e][l] += Wc[e][m] X[m][l]   — accumulated in registers over all m
//   P1 (K = l):  C[m][e] += X[m][l] Wr[e][l]   — reduced over the warps in shared memory and
//                over l-chunks by k_projm_sum in a fixed order (deterministic)
// Complex products use the 3-multiplication form (T1 = ar br, T2 = ai bi, T3 = (ar+ai)(br+bi)).
namespace {

__device__ __forceinline__ void dmma8(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
struct C3 {  // 3M accumulators of one 8x8 complex tile (2 values per thread)
  double t1[2], t2[2], t3[2];
  __device__ __forceinline__ void zero() { t1[0] = t1[1] = t2[0] = t2[1] = t3[0] = t3[1] = 0.0; }
  __device__ __forceinline__ void mma(double2 a, double2 b) {
    dmma8(t1[0], t1[1], a.x, b.x);
    dmma8(t2[0], t2[1], a.y, b.y);
    dmma8(t3[0], t3[1], a.x + a.y, b.x + b.y);
  }
  __device__ __forceinline__ double2 get(int h) const {
    return make_double2(t1[h] - t2[h], t3[h] - t1[h] - t2[h]);
  }
};

constexpr int PM_LC = 256, PM_LDX = PM_LC + 4;  // columns per CTA; padded row (== 4 mod 8)

template <int ET>
__global__ void __launch_bounds__(256) k_projm(ProjM P, Bufs bufs) {
  extern __shared__ __align__(16) double2 psm[];
  double2* Xs = psm;                    // [2][8][PM_LDX]
  double2* Wrs = Xs + 2 * 8 * PM_LDX;   // [8*ET][PM_LDX]
  double2* red = Wrs + 8 * ET * PM_LDX; // [NW][ET][8 m][8 e]
  const int lc = blockIdx.x, p = blockIdx.y;
  const int lb = P.l_begin + lc * PM_LC;  // this chunk's first column
  const int NW = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* X = reinterpret_cast<const double2*>(bufs.p[P.x_buf]) + P.x_off + (int64_t)p * P.nx * P.ny;
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  for (int c = threadIdx.x; c < 8 * ET * PM_LDX; c += blockDim.x) {
    const int e = c / PM_LDX, li = c % PM_LDX, l = lb + li;
    Wrs[c] = (e < P.E1 && li < PM_LC && l < P.l_end) ? TAB[P.wr + (int64_t)e * P.nx + l] : make_double2(0, 0);
  }
  const int ntile = (P.ny + 7) / 8;
  auto stage = [&](int it) {
    if (it < ntile) {
      double2* d = Xs + (it & 1) * 8 * PM_LDX;
      const int m0 = it * 8;
      for (int c = threadIdx.x; c < 8 * PM_LC; c += blockDim.x) {
        const int r = c / PM_LC, li = c % PM_LC, m = m0 + r, l = lb + li;
        const bool ok = m < P.ny && l < P.l_end;
        cp16p(d + r * PM_LDX + li, ok ? X + (int64_t)m * P.nx + l : X, ok);  // zero-fill outside
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  C3 h[ET][4];
#pragma unroll
  for (int et = 0; et < ET; ++et)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) h[et][nt].zero();
  const int lw = warp * 32;  // warp's columns within the chunk
  stage(0);
  for (int it = 0; it < ntile; ++it) {
    stage(it + 1);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    const double2* x = Xs + (it & 1) * 8 * PM_LDX;
    const int m0 = it * 8;
    // P2: C[e][l] += Wc[e][m] X[m][l]  (A = Wc 8e x 4m, B = X 4m x 8l)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int m = m0 + 4 * ks + q;
#pragma unroll
      for (int et = 0; et < ET; ++et) {
        const int e = et * 8 + g;
        const double2 a = (e < P.E2 && m < P.ny) ? __ldg(TAB + P.wc + (int64_t)e * P.ny + m) : make_double2(0, 0);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) h[et][nt].mma(a, x[(4 * ks + q) * PM_LDX + lw + 8 * nt + g]);
      }
    }
    // P1 partial: C[m][e] += X[m][l] Wr[e][l]  (A = X 8m x 4l, B = Wr^T 4l x 8e), K = warp's 32 l
    C3 gacc[ET];
#pragma unroll
    for (int et = 0; et < ET; ++et) gacc[et].zero();
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const double2 a = x[g * PM_LDX + lw + 4 * ks + q];
#pragma unroll
      for (int et = 0; et < ET; ++et) gacc[et].mma(a, Wrs[(et * 8 + g) * PM_LDX + lw + 4 * ks + q]);
    }
    // C fragment: thread holds C[m = g][e = 2q, 2q+1]
#pragma unroll
    for (int et = 0; et < ET; ++et)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) red[((warp * ET + et) * 8 + g) * 8 + 2 * q + hh] = gacc[et].get(hh);
    __syncthreads();
    for (int t = threadIdx.x; t < ET * 64; t += blockDim.x) {
      const int et = t / 64, m = m0 + (t / 8) % 8, e = et * 8 + t % 8;
      if (m < P.ny && e < P.E1) {
        double2 acc = make_double2(0, 0);
        for (int w = 0; w < NW; ++w) {
          const double2 v = red[((w * ET + et) * 8 + (t / 8) % 8) * 8 + t % 8];
          acc.x += v.x;
          acc.y += v.y;
        }
        IF[P.g_off + (int64_t)lc * P.g_lcs + (int64_t)e * P.g_es + (int64_t)p * P.g_ps + m] = acc;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // P2: thread holds C[e = et*8 + g][l = lw + 8nt + 2q (+1)]
#pragma unroll
  for (int et = 0; et < ET; ++et) {
    const int e = et * 8 + g;
    if (e >= P.E2) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int l = lb + lw + 8 * nt + 2 * q + hh;
        if (lw + 8 * nt + 2 * q + hh < PM_LC && l < P.l_end)
          IF[P.h_off + (int64_t)e * P.h_es + (int64_t)p * P.h_ps + l] = h[et][nt].get(hh);
      }
  }
}

// P1 = sum over l-chunks of the partials (fixed order)
__global__ void k_projm_sum(ProjM P, Bufs bufs) {
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  const int64_t n = (int64_t)P.E1 * P.nplanes * P.ny;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % P.ny);
    const int64_t rest = i / P.ny;
    const int p = (int)(rest % P.nplanes), e = (int)(rest / P.nplanes);
    double2 acc = make_double2(0, 0);
    for (int lc = 0; lc < P.nlc; ++lc) {
      const double2 v = IF[P.g_off + (int64_t)lc * P.g_lcs + (int64_t)e * P.g_es + (int64_t)p * P.g_ps + m];
      acc.x += v.x;
      acc.y += v.y;
    }
    IF[P.p1_off + (int64_t)e * P.p1_es + (int64_t)p * P.g_ps + m] = acc;
  }
}

}  // namespace

int projm_chunks(int nx) { return (nx + PM_LC - 1) / PM_LC; }

cudaError_t launch_projm(const ProjM& P, const Bufs& bufs, cudaStream_t st) {
  if (P.nplanes <= 0 || P.nplanes > 65535) return P.nplanes <= 0 ? cudaSuccess : cudaErrorInvalidValue;
  const int E = P.E1 > P.E2 ? P.E1 : P.E2;
  const int width = P.l_end - P.l_begin;
  if (width <= 0) return cudaSuccess;
  const int threads = width >= PM_LC ? PM_LC : ((width + 31) / 32) * 32;
  const int nw = threads / 32;
  const dim3 grid((unsigned)P.nlc, (unsigned)P.nplanes);
  cudaError_t e;
  if (E <= 8) {
    const size_t sm = (size_t)((2 * 8 + 8) * PM_LDX + nw * 64) * sizeof(double2);
    if ((e = cudaFuncSetAttribute(k_projm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    k_projm<1><<<grid, threads, sm, st>>>(P, bufs);
  } else if (E <= 16) {
    const size_t sm = (size_t)((2 * 8 + 16) * PM_LDX + nw * 128) * sizeof(double2);
    if ((e = cudaFuncSetAttribute(k_projm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    k_projm<2><<<grid, threads, sm, st>>>(P, bufs);
  } else {
    return cudaErrorInvalidValue;
  }
  if (P.nlc > 1 && P.E1 > 0) k_projm_sum<<<148 * 8, 256, 0, st>>>(P, bufs);
  return cudaGetLastError();
}

}  // namespace lfds
