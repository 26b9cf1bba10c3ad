// Step 5 of the blocked separable method in z-modal form.
//
// The global correction solves T_lm w^_lm = r^_lm for every global mode (l, m), with
// T_lm = A' + s_lm E, s_lm = lambda_l + mu_m (reading R1), and needs w only on the interface
// planes (P:56 last sentence; steps 6-7 take it from there).  When the z tables are real the
// pencil (A', E) has a real E-orthonormal eigenbasis Z (A' Z = E Z Theta, host setup), and
//   T_lm^{-1} = Z (Theta + s_lm)^{-1} Z^T.
// Transforming the small plane data to z-modes first (R~ = Z^T R, a real GEMM on the planes),
// the interface projections of w^ become, for every z-mode t,
//   C[m][l]   = sum_a R1~[a][t][m] W_x[I_a][l] + sum_b W_y[I_b][m] R2~[b][t][l]   (r^ of mode l,m,t)
//   Wh[m][l]  = C[m][l] / (mu_m + lambda_l + theta_t)                            (the z-solve)
//   P1~[a][t][m] = sum_l W_x[I_a][l] Wh[m][l],   P2~[b][t][l] = sum_m W_y[I_b][m] Wh[m][l]
// and P1 = Z P1~, P2 = Z P2~ (real GEMMs on the planes).  The N_x N_y N_z volume w^ is never
// stored: k_s5m streams (m, l) tiles through shared memory and keeps everything else on chip.
//
// k_s5m: one CTA per (r, t, 64-row m-tile), looping over 32-column l-tiles of this rank's
// x-modes.  Three DMMA (mma.sync.m8n8k4.f64) contractions per l-tile in the 3-multiplication
// complex form: C (K = |I|), P1 (K = l, accumulated in registers across the l loop, complete
// per CTA) and P2 (K = m over the tile: a partial per m-tile, summed by k_p2sum in a fixed
// order).  W_x / R2~ / lambda tiles are double-buffered with cp.async.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "lfds_internal.h"

namespace lfds {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpz16(void* dst, const void* src, bool valid) {  // zero-fill when !valid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// 3M accumulation of one complex 8x8x4 step: t1 += ar br, t2 += ai bi, t3 += (ar+ai)(br+bi)
__device__ __forceinline__ void cmma3(double (&t)[3][2], double2 a, double2 b) {
  dmma(t[0][0], t[0][1], a.x, b.x);
  dmma(t[1][0], t[1][1], a.y, b.y);
  dmma(t[2][0], t[2][1], a.x + a.y, b.x + b.y);
}
// 3M step with the A operand's (re, im, re + im) precomputed
__device__ __forceinline__ void cmma3s(double (&t)[3][2], double3 a, double2 b) {
  dmma(t[0][0], t[0][1], a.x, b.x);
  dmma(t[1][0], t[1][1], a.y, b.y);
  dmma(t[2][0], t[2][1], a.z, b.x + b.y);
}
// reciprocal from the MUFU.RCP64H seed and two Newton steps (full fp64 accuracy)
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double2 cres(const double (&t)[3][2], int h) {  // (re, im) of element h
  return make_double2(t[0][h] - t[1][h], t[2][h] - t[0][h] - t[1][h]);
}
__device__ __forceinline__ void zero3(double (&t)[3][2]) {
  t[0][0] = t[0][1] = t[1][0] = t[1][1] = t[2][0] = t[2][1] = 0.0;
}

constexpr int TM = 64, TL = 32, LW = TL + 1, LA = TM + 1, S5_THREADS = 256;

template <int KA>
struct S5Smem {
  static constexpr int WT = TM * LW;       // W^ tile [m][l]
  static constexpr int BX = KA * LW;       // W_x[I_a][l-tile], per buffer
  static constexpr int B2 = KA * LW;       // R2~[b][l-tile], per buffer
  static constexpr int LM = TL;            // lambda_l, per buffer
  static constexpr int A1 = KA * LA;       // R1~[a][m-tile]
  static constexpr int A2 = KA * LA;       // W_y[I_b][m-tile]
  static constexpr int CB = 4 * 64;        // phase-C half combine (KA = 8)
  static constexpr int TOTAL = WT + 2 * (BX + B2 + LM) + A1 + A2 + CB;
};

template <int KA>
__global__ void __launch_bounds__(S5_THREADS, KA <= 16 ? 2 : 1) k_s5m(S5M S, Bufs bufs) {
  static_assert(KA % 8 == 0 && KA <= 32, "KA: |I| padded to 8, 16 or 32");
  using SM = S5Smem<KA>;
  extern __shared__ __align__(16) double2 s5[];
  double2* Wt = s5;
  double2* Bx = Wt + SM::WT;
  double2* B2 = Bx + 2 * SM::BX;
  double2* LM = B2 + 2 * SM::B2;
  double2* A1 = LM + 2 * SM::LM;
  double2* A2 = A1 + SM::A1;
  double2* CB = A2 + SM::A2;
  const int mt = S.mt_begin + (int)blockIdx.x, t = blockIdx.y, r = blockIdx.z;
  const int m0 = mt * TM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  const int64_t rt = (int64_t)r * S.nz + t;  // merged (r, t) row of the plane arrays
  // ---- fixed operands of the CTA: R1~[a][rt][m-tile], W_y[I_b][m-tile] (zero outside)
  for (int c = tid; c < 2 * KA * TM; c += S5_THREADS) {
    const int which = c / (KA * TM), a = (c / TM) % KA, i = c % TM, m = m0 + i;
    if (which == 0)
      cpz16(A1 + a * LA + i, IF + S.r1t + ((int64_t)a * S.R * S.nz + rt) * S.ny + m, a < S.nifx && m < S.ny);
    else
      cpz16(A2 + a * LA + i, TAB + S.wyi + (int64_t)a * S.ny + m, a < S.nify && m < S.ny);
  }
  cp_commit();
  const int l_beg = S.l_begin, l_end = S.l_end;
  const int nlt = (l_end - l_beg + TL - 1) / TL;
  auto stage = [&](int lt) {
    if (lt < nlt) {
      const int l0 = l_beg + lt * TL, bf = lt & 1;
      for (int c = tid; c < 2 * KA * TL + TL; c += S5_THREADS) {
        if (c < KA * TL) {  // W_x[I_a][l]
          const int a = c / TL, j = c % TL, l = l0 + j;
          cpz16(Bx + bf * SM::BX + a * LW + j, TAB + S.wxi + (int64_t)a * S.nx + l, a < S.nifx && l < l_end);
        } else if (c < 2 * KA * TL) {  // R2~[b][rt][l]
          const int c2 = c - KA * TL, b = c2 / TL, j = c2 % TL, l = l0 + j;
          cpz16(B2 + bf * SM::B2 + b * LW + j, IF + S.r2t + ((int64_t)b * S.R * S.nz + rt) * S.nx + l,
                b < S.nify && l < l_end);
        } else {  // lambda_l
          const int j = c - 2 * KA * TL, l = l0 + j;
          cpz16(LM + bf * SM::LM + j, TAB + S.lamx + l, l < l_end);
        }
      }
    }
    cp_commit();
  };
  stage(0);
  cp_wait<1>();  // fixed operands
  __syncthreads();
  // A fragments of phase A for this warp's 8 rows m = 8 warp + g (fixed over the l loop)
  // (KA = 32: read from shared memory at each use instead, to stay within the register file)
  constexpr bool AREG = KA <= 16;
  constexpr int NFA = AREG ? KA / 4 : 1;
  double3 fa1[NFA], fa2[NFA];
  auto afrag = [&](const double2* Asm, int ks) {
    const double2 v = Asm[(4 * ks + q) * LA + 8 * warp + g];
    return make_double3(v.x, v.y, v.x + v.y);
  };
  if constexpr (AREG) {
#pragma unroll
    for (int ks = 0; ks < KA / 4; ++ks) {
      fa1[ks] = afrag(A1, ks);
      fa2[ks] = afrag(A2, ks);
    }
  }
  const int mrow = 8 * warp + g, mglob = m0 + mrow;
  const bool mok = mglob < S.ny;
  const double2 th = TAB[S.theta + t];
  double2 mu = mok ? TAB[S.lamy + mglob] : make_double2(0, 0);
  mu.x += th.x;
  mu.y += th.y;  // mu_m + theta_t
  // P1 accumulators: rows m = 8 warp + g, columns a = 8 as + 2q + h
  double p1[KA / 8][3][2];
#pragma unroll
  for (int as = 0; as < KA / 8; ++as) zero3(p1[as]);
  // phase-C assignment: (b-tile, l-tile) pairs over the warps, K = m split in halves if needed
  constexpr int NPAIR = (KA / 8) * 4, HALVES = NPAIR >= 8 ? 1 : 8 / NPAIR, KSC = TM / 4 / HALVES;
  constexpr int PSTEP = HALVES == 1 ? 8 : NPAIR;  // pairs of a warp: warp, warp + 8, ... (or one)
  const int pair0 = warp % NPAIR, half = HALVES == 1 ? 0 : warp / NPAIR;
  for (int lt = 0; lt < nlt; ++lt) {
    const int bf = lt & 1, l0 = l_beg + lt * TL;
    cp_wait<0>();
    __syncthreads();  // tile lt staged; tile lt-1 (W^ and its staging buffer) consumed
    stage(lt + 1);    // in flight while tile lt is computed
    const double2* bx = Bx + bf * SM::BX;
    const double2* b2 = B2 + bf * SM::B2;
    const double2* lm = LM + bf * SM::LM;
    {  // ---- phase A: C[m][l] for this warp's 8 rows and all 32 columns, then W^ = C / d
      double c[4][3][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) zero3(c[nt]);
#pragma unroll
      for (int ks = 0; ks < KA / 4; ++ks) {
        double3 x1, x2;
        if constexpr (AREG) {
          x1 = fa1[ks];
          x2 = fa2[ks];
        } else {
          x1 = afrag(A1, ks);
          x2 = afrag(A2, ks);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          cmma3s(c[nt], x1, bx[(4 * ks + q) * LW + 8 * nt + g]);
          cmma3s(c[nt], x2, b2[(4 * ks + q) * LW + 8 * nt + g]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 8 * nt + 2 * q + h;
          const double2 cv = cres(c[nt], h), la = lm[j];
          const double dr = mu.x + la.x, di = mu.y + la.y;
          const double inv = fast_rcp(fma(dr, dr, di * di));
          double2 w = make_double2(fma(cv.x, dr, cv.y * di) * inv, fma(cv.y, dr, -cv.x * di) * inv);
          if (!mok || l0 + j >= l_end) w = make_double2(0, 0);
          Wt[mrow * LW + j] = w;
        }
    }
    __syncthreads();  // W^ tile complete
    // ---- phase B: P1[m][a] += sum_l W^[m][l] W_x[I_a][l] (rows m = this warp's 8)
#pragma unroll
    for (int ks = 0; ks < TL / 4; ++ks) {
      const double2 aw = Wt[mrow * LW + 4 * ks + q];
#pragma unroll
      for (int as = 0; as < KA / 8; ++as) cmma3(p1[as], aw, bx[(8 * as + g) * LW + 4 * ks + q]);
    }
    // ---- phase C: P2 partial[b][l] = sum_{m in tile} W_y[I_b][m] W^[m][l]
#pragma unroll
    for (int pair = pair0; pair < NPAIR; pair += PSTEP) {
      const int cbs = pair / 4, cls = pair % 4;
      double p2[3][2];
      zero3(p2);
#pragma unroll
      for (int ks = 0; ks < KSC; ++ks) {
        const int mm = (half * KSC + ks) * 4 + q;
        cmma3(p2, A2[(8 * cbs + g) * LA + mm], Wt[mm * LW + 8 * cls + g]);
      }
      const int b = 8 * cbs + g;
      if (HALVES == 2) {
        if (half == 1) {
#pragma unroll
          for (int h = 0; h < 2; ++h) CB[pair * 64 + lane * 2 + h] = cres(p2, h);
        }
        __syncthreads();
      }
      if (half == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 v = cres(p2, h);
          if (HALVES == 2) {
            const double2 o = CB[pair * 64 + lane * 2 + h];
            v.x += o.x;
            v.y += o.y;
          }
          const int l = l0 + 8 * cls + 2 * q + h;
          if (b < S.nify && l < l_end)
            IF[S.p2p + (((int64_t)b * S.R * S.nz + rt) * S.nmt + mt) * S.nx + l] = v;
        }
      }
    }
  }
  cp_wait<0>();
  // ---- P1~[a][rt][m] (complete over this rank's x-modes)
  if (mok) {
#pragma unroll
    for (int as = 0; as < KA / 8; ++as)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * as + 2 * q + h;
        if (a < S.nifx) IF[S.p1t + ((int64_t)a * S.R * S.nz + rt) * S.ny + mglob] = cres(p1[as], h);
      }
  }
}

// P2~[b][rt][l] = sum over the m-tiles of the partials (fixed order); zero outside [l_begin, l_end)
__global__ void k_p2sum(S5M S, Bufs bufs) {
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  const int64_t rows = (int64_t)S.nify * S.R * S.nz, n = rows * S.nx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / S.nx;
    const int l = (int)(i - row * S.nx);
    double2 acc = make_double2(0, 0);
    if (l >= S.l_begin && l < S.l_end) {
      const double2* p = IF + S.p2p + row * S.nmt * S.nx + l;
      for (int k = S.mt_begin; k < S.mt_end; ++k) {
        const double2 v = p[(int64_t)k * S.nx];
        acc.x += v.x;
        acc.y += v.y;
      }
    }
    IF[S.p2t + i] = acc;
  }
}

}  // namespace

int s5m_ka(int nifx, int nify) {
  const int n = nifx > nify ? nifx : nify;
  return n <= 8 ? 8 : n <= 16 ? 16 : n <= 32 ? 32 : 0;
}
int s5m_mtiles(int ny) { return (ny + TM - 1) / TM; }

cudaError_t launch_s5m(const S5M& S, const Bufs& bufs, cudaStream_t st) {
  const int ka = s5m_ka(S.nifx, S.nify);
  if (!ka || S.R > 65535 || S.nz > 65535) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)(S.mt_end - S.mt_begin), (unsigned)S.nz, (unsigned)S.R);
  cudaError_t e;
  if (S.mt_end > S.mt_begin) {  // (a rank without x-modes still writes P1~ = 0 on its m rows)
    if (ka == 8) {
      const size_t sm = S5Smem<8>::TOTAL * sizeof(double2);
      if ((e = cudaFuncSetAttribute(k_s5m<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
      k_s5m<8><<<grid, S5_THREADS, sm, st>>>(S, bufs);
    } else if (ka == 16) {
      const size_t sm = S5Smem<16>::TOTAL * sizeof(double2);
      if ((e = cudaFuncSetAttribute(k_s5m<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
      k_s5m<16><<<grid, S5_THREADS, sm, st>>>(S, bufs);
    } else {
      const size_t sm = S5Smem<32>::TOTAL * sizeof(double2);
      if ((e = cudaFuncSetAttribute(k_s5m<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
      k_s5m<32><<<grid, S5_THREADS, sm, st>>>(S, bufs);
    }
    if ((e = cudaGetLastError())) return e;
  }
  if (S.nify > 0) {
    const int64_t n = (int64_t)S.nify * S.R * S.nz * S.nx;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_p2sum<<<(unsigned)blocks, 256, 0, st>>>(S, bufs);
  }
  return cudaGetLastError();
}

}  // namespace lfds
