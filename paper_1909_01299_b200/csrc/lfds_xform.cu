// Block transform passes on the FP64 tensor pipe (DMMA, mma.sync.m8n8k4.f64 -> SASS DMMA.8).
//
// Steps 1 and 7 of PAPER.md:66/:72 apply a small n x n eigenvector matrix S (F = W^T M
// forward, W inverse) along x or along y of every block:
//     C(i, n) = sum_j S(i, j) B(j, n)                          (GemmDesc addressing)
// with S in the plan tables and B, C the data (n = every other index of the block).
// sm_100a has no tcgen05 kind for f64, so the tensor path is the legacy warp-level DMMA
// (8x8x4, one double per thread for A and B); on B200 it runs at the same 37 TF/s as DFMA
// (profiles/r01_fp64_peaks.log) but with 8x fewer issued instructions per FMA.
//
//  * complex S (C blocks): 4 real MMAs per complex 8x8x4 step (re*re - im*im, re*im + im*re)
//  * real S (U, R blocks; also exact sine modes): the complex data is viewed as a real matrix
//    with interleaved (re, im) columns, so C = S B is ONE real GEMM — half the flops.
// Tiles: CTA 64 (S rows) x 64 (complex data columns), K chunks of 16 double-buffered in
// shared memory with cp.async (16-byte copies, zero-fill outside the ragged edges).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "lfds_internal.h"

namespace lfds {

namespace {

constexpr int XT_M = 64, XT_N = 64, XT_K = 16, XT_THREADS = 128;
constexpr int LDA_C = XT_M + 2;   // complex A tile row stride (16-B units) == 2 mod 8
constexpr int LDA_R = XT_M + 4;   // real A tile row stride (8-B units) == 4 mod 16
constexpr int LDB_C = XT_N + 2;   // complex B tile row stride == 2 mod 8 (real view 2*LDB_C == 4 mod 16)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// (n1, n2) of column n + step from those of column n (n = n1 * N2 + n2), with the step's own
// decomposition step = d1 * N2 + d2 precomputed once per thread (no division per column)
struct ColStep {
  int d1, d2;  // step <= 16, so both fit 32 bits
  __device__ __forceinline__ ColStep(int step, int64_t N2)
      : d1((int)(step / N2)), d2((int)(step - (step / N2) * N2)) {}
  __device__ __forceinline__ void advance(int64_t& n1, int64_t& n2, int64_t N2) const {
    n1 += d1;
    n2 += d2;
    if (n2 >= N2) { n2 -= N2; ++n1; }
  }
};

template <bool REAL_S>
struct XSmem {
  static constexpr int A_ELEMS = REAL_S ? XT_K * LDA_R : XT_K * LDA_C * 2;  // in doubles
  static constexpr int B_ELEMS = XT_K * LDB_C * 2;                          // in doubles
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = (size_t)2 * STAGE * sizeof(double);
};

// SMALLM (real S, M <= 32: blocks of at most 32 nodes): a 32-row tile, every warp 32 rows x
// 16 complex columns, so no warp works on the all-zero rows 32..63 of the 64-row tile.
template <bool REAL_S, bool KCONTIG, bool SMALLM = false>
// min blocks: 3 CTAs per SM for the 64-row tiles (168 registers instead of 194: C4q step-5 z-transforms
// 1.23 -> 1.17 ms), 4 for SMALLM (its 116-128 registers unchanged)
__global__ void __launch_bounds__(XT_THREADS, SMALLM ? 4 : 3) k_xform(const GemmDesc* __restrict__ descs, int gm, Bufs bufs) {
  static_assert(REAL_S || !SMALLM, "SMALLM: real S only");
  constexpr int TM = SMALLM ? 32 : XT_M;
  constexpr int NJ = SMALLM ? 4 : 8;  // real-view 8-column tiles per warp
  extern __shared__ __align__(16) double xsm[];
  __shared__ GemmDesc sD;  // (see k_xform3m: global-memory descriptor fields are re-read after barriers)
  if (threadIdx.x < (int)(sizeof(GemmDesc) / 8))
    reinterpret_cast<int64_t*>(&sD)[threadIdx.x] = reinterpret_cast<const int64_t*>(descs + blockIdx.z)[threadIdx.x];
  __syncthreads();
  const GemmDesc& D = sD;
  const int M = D.M, K = D.K;
  const int64_t N2 = D.N2, N = (int64_t)D.N1 * D.N2;
  // row tiles fastest: the CTAs of one column tile run together and share its B tile in L2
  const int i0 = (int)(blockIdx.x % gm) * TM;
  const int64_t n0 = (int64_t)(blockIdx.x / gm) * XT_N;
  if (i0 >= M || n0 >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp tile origin (row, complex column)
  const int wm = SMALLM ? 0 : (warp >> 1) * 32, wn = SMALLM ? warp * 16 : (warp & 1) * 32;
  const int g = lane >> 2, q = lane & 3;

  const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off;
  // ---- per-thread load assignments (fixed across K chunks)
  // A (S): TM x 16 elements, thread -> row ai = tid/2, 8 consecutive j (SMALLM: tid/4, 4 j)
  constexpr int AJ = SMALLM ? 4 : 8;
  const int ai = SMALLM ? tid >> 2 : tid >> 1, aj0 = SMALLM ? (tid & 3) * 4 : (tid & 1) * 8;
  const bool arow_ok = (i0 + ai) < M;
  // B (data): 16 x 64 complex.  Coalesced mappings: K-contiguous data -> 16 threads cover
  // one 256-byte column segment (8 columns per instruction); otherwise 64 consecutive
  // threads cover 64 consecutive columns of one row (2 rows per instruction).
  int64_t bcol[8];
  int bj, bn0;
  if (KCONTIG) {  // thread -> j = tid % 16, columns tid/16 + 8e
    bj = tid & 15;
    bn0 = tid >> 4;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t n = n0 + bn0 + 8 * e;
      const int64_t n1 = n / N2, n2 = n - n1 * N2;
      bcol[e] = (n < N) ? n1 * D.sB1 + n2 * D.sB2 : -1;
    }
  } else {        // thread -> column tid % 64, rows tid/64 + 2e
    bj = tid >> 6;
    bn0 = tid & 63;
    const int64_t n = n0 + bn0;
    const int64_t n1 = n / N2, n2 = n - n1 * N2;
    bcol[0] = (n < N) ? n1 * D.sB1 + n2 * D.sB2 : -1;
  }

  auto load_chunk = [&](int stage, int j0) {
    double* As = xsm + stage * XSmem<REAL_S>::STAGE;
    double2* Bs = reinterpret_cast<double2*>(As + XSmem<REAL_S>::A_ELEMS);
    if (REAL_S) {
      const double* A = reinterpret_cast<const double*>(bufs.p[B_TAB]) + D.a_off;
#pragma unroll
      for (int e = 0; e < AJ; ++e) {
        const int j = j0 + aj0 + e;
        const bool ok = arow_ok && j < K;
        cp_async8(As + (aj0 + e) * LDA_R + ai, ok ? A + (int64_t)(i0 + ai) * D.sAi + (int64_t)j * D.sAj : A, ok);
      }
    } else {
      const double2* A = reinterpret_cast<const double2*>(bufs.p[B_TAB]) + D.a_off;
      double2* As2 = reinterpret_cast<double2*>(As);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = j0 + aj0 + e;
        const bool ok = arow_ok && j < K;
        cp_async16(As2 + (aj0 + e) * LDA_C + ai, ok ? A + (int64_t)(i0 + ai) * D.sAi + (int64_t)j * D.sAj : A, ok);
      }
    }
    if (KCONTIG) {
      const int j = j0 + bj;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = bcol[e] >= 0 && j < K;
        cp_async16(Bs + bj * LDB_C + bn0 + 8 * e, ok ? B + bcol[e] + j : B, ok);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = j0 + bj + 2 * e;
        const bool ok = bcol[0] >= 0 && j < K;
        cp_async16(Bs + (bj + 2 * e) * LDB_C + bn0, ok ? B + bcol[0] + (int64_t)j * D.sBj : B, ok);
      }
    }
  };

  // accumulators: complex S -> [4 row tiles][4 col tiles][re/im][2]; real S -> [4][8][2] over
  // the real view (8 real column tiles of 8 = 32 complex columns)
  double acc[4][NJ][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NJ; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int nchunks = (K + XT_K - 1) / XT_K;
  load_chunk(0, 0);
  cp_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) load_chunk((c + 1) & 1, (c + 1) * XT_K);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* As = xsm + (c & 1) * XSmem<REAL_S>::STAGE;
    const double* Bs = As + XSmem<REAL_S>::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < XT_K; kk += 4) {
      if (REAL_S) {
        double a[4], b[NJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[(kk + q) * LDA_R + wm + 8 * i + g];
#pragma unroll
        for (int j = 0; j < NJ; ++j) b[j] = Bs[(kk + q) * (2 * LDB_C) + 2 * wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      } else {
        const double2* As2 = reinterpret_cast<const double2*>(As);
        const double2* Bs2 = reinterpret_cast<const double2*>(Bs);
        double2 a[4], b[4];
        static_assert(NJ == 8 || REAL_S, "complex S uses the 64 x 64 tile");
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As2[(kk + q) * LDA_C + wm + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs2[(kk + q) * LDB_C + wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double nai = -a[i].y;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // acc[i][2j] = re part, acc[i][2j+1] = im part
            dmma(acc[i][2 * j][0], acc[i][2 * j][1], a[i].x, b[j].x);
            dmma(acc[i][2 * j][0], acc[i][2 * j][1], nai, b[j].y);
            dmma(acc[i][2 * j + 1][0], acc[i][2 * j + 1][1], a[i].x, b[j].y);
            dmma(acc[i][2 * j + 1][0], acc[i][2 * j + 1][1], a[i].y, b[j].x);
          }
        }
      }
    }
    __syncthreads();
  }
  cp_wait<0>();

  // ---- epilogue: thread holds C rows (wm + 8i + g), columns 2q, 2q+1 of each 8-wide tile.
  // Columns outer, rows inner: a column's offset is stepped from the previous one (one 64-bit
  // division per thread, not one per stored element).
  double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off;
  {
    // columns in store order: real S -> wn + 4j + q (j < 8); complex S -> wn + 8j' + 2q + h
    int64_t n = n0 + wn + (REAL_S ? q : 2 * q);
    int64_t n1 = n / N2, n2 = n - n1 * N2;
    const ColStep c1(1, N2), c4(4, N2), c7(7, N2);
#pragma unroll
    for (int e = 0; e < NJ; ++e) {
      if (n < N) {
        const int64_t off = n1 * D.sC1 + n2 * D.sC2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i0 + wm + 8 * i + g;
          if (row >= M) continue;
          // real S: acc[i][e] = (re, im) of column e; complex S: re in acc[i][2j], im in acc[i][2j+1]
          const double2 v = REAL_S ? make_double2(acc[i][e][0], acc[i][e][1])
                                   : make_double2(acc[i][(2 * (e >> 1)) % NJ][e & 1], acc[i][(2 * (e >> 1) + 1) % NJ][e & 1]);
          C[(int64_t)row * D.sCi + off] = v;
        }
      }
      if (REAL_S) { n += 4; c4.advance(n1, n2, N2); }
      else if (e & 1) { n += 7; c7.advance(n1, n2, N2); }
      else { n += 1; c1.advance(n1, n2, N2); }
    }
  }
}

template <bool REAL_S, bool KCONTIG, bool SMALLM>
cudaError_t launch_one_t(const GemmDesc* d, int ndesc, int maxM, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  const size_t sm = XSmem<REAL_S>::BYTES;
  constexpr int TM = SMALLM ? 32 : XT_M;
  cudaError_t e = cudaFuncSetAttribute(k_xform<REAL_S, KCONTIG, SMALLM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  for (int z0 = 0; z0 < ndesc; z0 += 65535) {
    const int nzz = ndesc - z0 < 65535 ? ndesc - z0 : 65535;
    const int gm = (maxM + TM - 1) / TM;
    dim3 grid((unsigned)(((maxN + XT_N - 1) / XT_N) * gm), 1, (unsigned)nzz);
    k_xform<REAL_S, KCONTIG, SMALLM><<<grid, XT_THREADS, sm, st>>>(d + z0, gm, bufs);
  }
  return cudaGetLastError();
}
template <bool REAL_S, bool KCONTIG>
cudaError_t launch_one(const GemmDesc* d, int ndesc, int maxM, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  if (REAL_S && maxM <= 32) return launch_one_t<true, KCONTIG, true>(d, ndesc, maxM, maxN, bufs, st);
  return launch_one_t<REAL_S, KCONTIG, false>(d, ndesc, maxM, maxN, bufs, st);
}


// ---------------------------------------------------------------- persistent small real-S form
// Blocks of at most 32 nodes with a real basis (R / U blocks of C3, C5): S is at most 32 x 32, so
// k_xform's CTAs were short (two K chunks of 16, then the epilogue) and re-staged S per 64-column
// tile.  k_xsmall keeps S in shared memory for the CTA's life and streams its column tiles (all K
// rows of 64 complex columns at once) through a three-stage cp.async ring: two tiles in flight
// while one is contracted.  Same warp tiling (32 rows x 16 complex columns per warp), arithmetic
// order and epilogue as k_xform<true, *, true>, so the result is bit-identical.
template <int KS>
struct XsSmem {
  static constexpr int NST = 3;
  static constexpr int LDA = 36;                  // S rows (<= 32) padded, == 4 mod 16
  static constexpr int A = KS * LDA;              // doubles
  static constexpr int B = KS * LDB_C * 2;        // doubles per stage
  static constexpr size_t BYTES = (size_t)(A + NST * B) * sizeof(double);
};

template <bool KCONTIG, int KS>
__global__ void __launch_bounds__(XT_THREADS, 2) k_xsmall(const GemmDesc* __restrict__ descs, Bufs bufs) {
  using SM = XsSmem<KS>;
  constexpr int NST = SM::NST, NJ = 4;
  extern __shared__ __align__(16) double xsm[];
  __shared__ GemmDesc sD;
  if (threadIdx.x < (int)(sizeof(GemmDesc) / 8))
    reinterpret_cast<int64_t*>(&sD)[threadIdx.x] = reinterpret_cast<const int64_t*>(descs + blockIdx.y)[threadIdx.x];
  __syncthreads();
  const GemmDesc& D = sD;
  const int M = D.M, K = D.K;
  const int64_t N2 = D.N2, N = (int64_t)D.N1 * D.N2;
  const int64_t ntiles = (N + XT_N - 1) / XT_N;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp * 16, g = lane >> 2, q = lane & 3;
  double* As = xsm;
  double* Bsm = xsm + SM::A;
  {  // S once: As[j][i] = S(i, j), zero outside M x K
    const double* A = reinterpret_cast<const double*>(bufs.p[B_TAB]) + D.a_off;
    for (int c = tid; c < KS * 32; c += XT_THREADS) {
      const int j = c >> 5, i = c & 31;
      As[j * SM::LDA + i] = (i < M && j < K) ? __ldg(A + (int64_t)i * D.sAi + (int64_t)j * D.sAj) : 0.0;
    }
  }
  const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off;
  const int bj = KCONTIG ? (tid & 15) : (tid >> 6), bn0 = KCONTIG ? (tid >> 4) : (tid & 63);
  const ColStep c8(8, N2);
  auto issue = [&](int64_t t, int stage) {
    if (t < ntiles) {
      double2* Bs = reinterpret_cast<double2*>(Bsm + stage * SM::B);
      if (KCONTIG) {  // 16 threads per 256-byte column segment, columns bn0 + 8e
        int64_t n = t * XT_N + bn0;
        int64_t n1 = n / N2, n2 = n - n1 * N2;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool nok = n < N;
          const int64_t col = n1 * D.sB1 + n2 * D.sB2;
#pragma unroll
          for (int h = 0; h < KS / 16; ++h) {
            const int j = bj + 16 * h;
            const bool ok = nok && j < K;
            cp_async16(Bs + j * LDB_C + bn0 + 8 * e, ok ? B + col + j : B, ok);
          }
          n += 8;
          c8.advance(n1, n2, N2);
        }
      } else {  // 64 consecutive columns of one row per 64 threads, rows bj + 2e
        const int64_t n = t * XT_N + bn0;
        const int64_t n1 = n / N2, n2 = n - n1 * N2;
        const int64_t col = n1 * D.sB1 + n2 * D.sB2;
#pragma unroll
        for (int e = 0; e < KS / 2; ++e) {
          const int j = bj + 2 * e;
          const bool ok = n < N && j < K;
          cp_async16(Bs + j * LDB_C + bn0, ok ? B + col + (int64_t)j * D.sBj : B, ok);
        }
      }
    }
    cp_commit();
  };
  const int64_t G = gridDim.x;
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) issue(blockIdx.x + s * G, s);
  double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off;
  const ColStep c1(1, N2), c4(4, N2);
  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G, ++k) {
    __syncthreads();  // stage (k - 1) % NST read by every warp before it is refilled
    issue(t + (NST - 1) * G, (k + NST - 1) % NST);
    cp_wait<NST - 1>();
    __syncthreads();  // tile t landed for every thread
    const double* Bs = Bsm + (k % NST) * SM::B;
    double acc[4][NJ][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < NJ; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KS; kk += 4) {
      double a[4], b[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(kk + q) * SM::LDA + 8 * i + g];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = Bs[(kk + q) * (2 * LDB_C) + 2 * wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    // epilogue (k_xform's real-S order): columns wn + 4j + q, rows 8i + g
    int64_t n = t * XT_N + wn + q;
    int64_t n1 = n / N2, n2 = n - n1 * N2;
#pragma unroll
    for (int e = 0; e < NJ; ++e) {
      if (n < N) {
        const int64_t off = n1 * D.sC1 + n2 * D.sC2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = 8 * i + g;
          if (row < M) C[(int64_t)row * D.sCi + off] = make_double2(acc[i][e][0], acc[i][e][1]);
        }
      }
      n += 4;
      c4.advance(n1, n2, N2);
    }
  }
  cp_wait<0>();
}

template <bool KCONTIG, int KS>
cudaError_t launch_xsmall_t(const GemmDesc* d, int ndesc, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  const size_t sm = XsSmem<KS>::BYTES;
  auto kern = k_xsmall<KCONTIG, KS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, XT_THREADS, sm)) != cudaSuccess) return e;
  const int64_t ntiles = (maxN + XT_N - 1) / XT_N;
  for (int y0 = 0; y0 < ndesc; y0 += 65535) {
    const int ny = ndesc - y0 < 65535 ? ndesc - y0 : 65535;
    // persistent CTAs over all descriptors of the launch, a whole number of waves (equal CTAs:
    // a partial last wave would leave SMs idle for a whole CTA lifetime); else many waves
    const int64_t cap = (int64_t)std::max(1, per) * sms;
    int64_t per_desc = 0;
    for (int64_t p = std::max<int64_t>(1, cap / ny); p <= std::max<int64_t>(1, 16 * cap / ny); ++p)
      if ((p * ny) % cap == 0) { per_desc = p; break; }
    if (!per_desc) per_desc = std::max<int64_t>(1, 16 * cap / ny);
    per_desc = std::min<int64_t>(per_desc, ntiles);
    kern<<<dim3((unsigned)per_desc, (unsigned)ny), XT_THREADS, sm, st>>>(d + y0, bufs);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- plane form, both bases real
// Blocks whose x AND y bases are real and at most 32 nodes long (the R x R blocks of C5 / C3):
// steps 1 and 7 as ONE pass over the block instead of an x pass and a y pass,
//   Out[m][l] = sum_q Ay[m][q] T[q][l],   T[q][l] = sum_p In[q][p] Ax[l][p],
// with the x-transformed plane T kept in shared memory (32 B per element of HBM traffic per
// direction instead of 64).  A CTA owns one block (Ax, Ay staged once, K-major like k_xsmall)
// and streams its planes through a cp.async ring (two stages at three CTAs per SM); per plane two DMMA phases with
// the complex data viewed as real (re, im) columns:
//   phase 1: rows l (Ax as the A operand), columns (q, re/im): warp w takes q = 4w .. 4w + 3;
//   phase 2: rows m (Ay),                  columns (l, re/im): warp w takes l = 4w .. 4w + 3.
// Same K order (p, q ascending in steps of 4) and DMMA shapes as the two k_xsmall passes, so
// the result is bit-identical to theirs.  The output is staged in the consumed input buffer and
// stored by rows (coalesced).  Strides: In rows 36 units (B fragments of phase 1 conflict-free:
// 2 * 36 == 8 mod 16), T rows 34 (phase-2 B fragments: 2 * 34 == 4 mod 16; phase-1 stores hit
// four 32-B bank groups).
constexpr int XP_THREADS = 256, XP_LDA = 36, XP_LDI = 36, XP_LDT = 34;
// A complex basis on an axis (CX / CY: C blocks of at most 32 nodes next to the real ones, and
// C x C corner blocks) takes a second real matrix Im A and a second DMMA per step against the
// data with its (re, im) slots swapped and the re slot negated:
//   (Ar + i Ai)(Br + i Bi):  re = Ar Br + Ai (-Bi),  im = Ar Bi + Ai Br.
template <int XP_NST, bool CX, bool CY>
constexpr size_t xp_bytes() {
  return (size_t)((2 + CX + CY) * 32 * XP_LDA + 2 * (XP_NST * 32 * XP_LDI + 32 * XP_LDT)) * sizeof(double);
}

template <int XP_NST, int MINB, bool CX, bool CY>
__global__ void __launch_bounds__(XP_THREADS, MINB) k_xplane(const XPlaneDesc* __restrict__ descs, Bufs bufs) {
  extern __shared__ __align__(16) double xsm[];
  __shared__ XPlaneDesc sD;
  static_assert(sizeof(XPlaneDesc) % 8 == 0, "descriptor copied as 64-bit words");
  if (threadIdx.x < (int)(sizeof(XPlaneDesc) / 8))
    reinterpret_cast<int64_t*>(&sD)[threadIdx.x] = reinterpret_cast<const int64_t*>(descs + blockIdx.y)[threadIdx.x];
  __syncthreads();
  const XPlaneDesc& D = sD;
  const int nx = D.nx, ny = D.ny, np = D.nplanes;
  if ((int)blockIdx.x >= np) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  double* AsX = xsm;                   // AsX[p][l] = Ax(l, p)
  double* AsY = xsm + 32 * XP_LDA;     // AsY[q][m] = Ay(m, q)
  double* AsXi = xsm + 2 * 32 * XP_LDA;              // imaginary parts (CX / CY)
  double* AsYi = xsm + (2 + CX) * 32 * XP_LDA;
  double2* Ins = reinterpret_cast<double2*>(xsm + (2 + CX + CY) * 32 * XP_LDA);  // [NST][32][LDI]
  double2* Ts = Ins + XP_NST * 32 * XP_LDI;                          // [32][LDT]: T[q][l]
  {
    const double* TABd = reinterpret_cast<const double*>(bufs.p[B_TAB]);
    for (int c = tid; c < 32 * 32; c += XP_THREADS) {
      const int i = c >> 5, j = c & 31;  // (out, in)
      const double2* TABz = reinterpret_cast<const double2*>(TABd);  // complex matrices: offsets in complex units
      if constexpr (CX) {
        const double2 z = (i < nx && j < nx) ? __ldg(TABz + D.ax + (int64_t)i * nx + j) : make_double2(0.0, 0.0);
        AsX[j * XP_LDA + i] = z.x;
        AsXi[j * XP_LDA + i] = z.y;
      } else {
        AsX[j * XP_LDA + i] = (i < nx && j < nx) ? __ldg(TABd + D.ax + (int64_t)i * nx + j) : 0.0;
      }
      if constexpr (CY) {
        const double2 z = (i < ny && j < ny) ? __ldg(TABz + D.ay + (int64_t)i * ny + j) : make_double2(0.0, 0.0);
        AsY[j * XP_LDA + i] = z.x;
        AsYi[j * XP_LDA + i] = z.y;
      } else {
        AsY[j * XP_LDA + i] = (i < ny && j < ny) ? __ldg(TABd + D.ay + (int64_t)i * ny + j) : 0.0;
      }
    }
  }
  const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off;
  double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off;
  // plane r into ring slot `stage`: 32 x 32 slots, zero outside ny x nx (a lane per column)
  auto issue = [&](int r, int stage) {
    if (r < np) {
      double2* dst = Ins + stage * 32 * XP_LDI;
      const double2* src = B + (int64_t)r * D.sB1;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = (tid >> 5) + 8 * e, col = lane;
        const bool ok = row < ny && col < nx;
        cp_async16(dst + row * XP_LDI + col, ok ? src + (int64_t)row * D.sBr + col : B, ok);
      }
    }
    cp_commit();
  };
  const int G = gridDim.x;
  const double sgn = (g & 1) ? 1.0 : -1.0;  // swapped-slot operand of a complex basis: (-Bi, Br)
#pragma unroll
  for (int s = 0; s < XP_NST - 1; ++s) issue((int)blockIdx.x + s * G, s);
  int k = 0;
  for (int r = blockIdx.x; r < np; r += G, ++k) {
    __syncthreads();  // slot (k - 1) % NST stored out by every thread before it is refilled
    issue(r + (XP_NST - 1) * G, (k + XP_NST - 1) % XP_NST);
    cp_wait<XP_NST - 1>();
    __syncthreads();  // plane r landed for every thread (and AsX / AsY on the first plane)
    double2* In = Ins + (k % XP_NST) * 32 * XP_LDI;
    double acc[4][2];
    {  // ---- phase 1: T[q][l], rows l = 8i + g, complex column q = 4 warp + (lane & 3)
      const double* Ind = reinterpret_cast<const double*>(In);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = AsX[(kk + q) * XP_LDA + 8 * i + g];
        const int ad = ((4 * warp + (g >> 1)) * XP_LDI + kk + q) * 2 + (g & 1);
        const double b = Ind[ad];
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], a[i], b);
        if constexpr (CX) {
          const double bp = sgn * Ind[ad ^ 1];
#pragma unroll
          for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], AsXi[(kk + q) * XP_LDA + 8 * i + g], bp);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) Ts[(4 * warp + q) * XP_LDT + 8 * i + g] = make_double2(acc[i][0], acc[i][1]);
    }
    __syncthreads();  // T complete; the input plane is consumed
    {  // ---- phase 2: Out[m][l], rows m = 8i + g, complex column l = 4 warp + (lane & 3)
      const double* Td = reinterpret_cast<const double*>(Ts);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = AsY[(kk + q) * XP_LDA + 8 * i + g];
        const int ad = (kk + q) * (2 * XP_LDT) + 8 * warp + g;
        const double b = Td[ad];
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], a[i], b);
        if constexpr (CY) {
          const double bp = sgn * Td[ad ^ 1];
#pragma unroll
          for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], AsYi[(kk + q) * XP_LDA + 8 * i + g], bp);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) In[(8 * i + g) * XP_LDI + 4 * warp + q] = make_double2(acc[i][0], acc[i][1]);
    }
    __syncthreads();  // output plane staged (and T consumed)
    double2* dst = C + (int64_t)r * D.sC1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = (tid >> 5) + 8 * e, col = lane;
      if (row < ny && col < nx) dst[(int64_t)row * D.sCr + col] = In[row * XP_LDI + col];
    }
  }
  cp_wait<0>();
}

}  // namespace

// plane transforms of blocks with two real bases of at most 32 nodes: persistent CTAs per block,
// a whole number of waves over the launch (see launch_xsmall_t)
template <class K>
static cudaError_t launch_xplane_k(K kern, int threads, size_t sm, int planes_per_cta_iter, const XPlaneDesc* d,
                                   int ndesc, int nplanes, const Bufs& bufs, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, sm)) != cudaSuccess) return e;
  const int64_t items = (nplanes + planes_per_cta_iter - 1) / planes_per_cta_iter;
  for (int y0 = 0; y0 < ndesc; y0 += 65535) {
    const int ny = ndesc - y0 < 65535 ? ndesc - y0 : 65535;
    const int64_t cap = (int64_t)std::max(1, per) * sms;
    int64_t per_desc = 0;
    for (int64_t p = std::max<int64_t>(1, cap / ny); p <= std::max<int64_t>(1, 16 * cap / ny); ++p)
      if ((p * ny) % cap == 0) { per_desc = p; break; }
    if (!per_desc) per_desc = std::max<int64_t>(1, 16 * cap / ny);
    per_desc = std::min<int64_t>(per_desc, items);
    kern<<<dim3((unsigned)per_desc, (unsigned)ny), threads, sm, st>>>(d + y0, bufs);
  }
  return cudaGetLastError();
}

// mode 1 (default): a two-stage ring at three CTAs per SM (73 KB each); 4: a three-stage ring at two
// CTAs per SM (A/B: 97.3 vs 95.7 ms per C5 step for mode 1, profiles/r02/xplane_modes).  cx / cy: the
// basis of that axis is complex (offsets ax / ay in complex units); those forms run two CTAs per SM.
cudaError_t launch_xplane(const XPlaneDesc* d, int ndesc, int nplanes, const Bufs& bufs, cudaStream_t st, int mode,
                          bool cx, bool cy) {
  if (ndesc <= 0 || nplanes <= 0) return cudaSuccess;
  if (cx && cy)
    return launch_xplane_k(k_xplane<2, 2, true, true>, XP_THREADS, xp_bytes<2, true, true>(), 1, d, ndesc, nplanes, bufs, st);
  if (cx)
    return launch_xplane_k(k_xplane<2, 2, true, false>, XP_THREADS, xp_bytes<2, true, false>(), 1, d, ndesc, nplanes, bufs, st);
  if (cy)
    return launch_xplane_k(k_xplane<2, 2, false, true>, XP_THREADS, xp_bytes<2, false, true>(), 1, d, ndesc, nplanes, bufs, st);
  if (mode == 4)
    return launch_xplane_k(k_xplane<3, 2, false, false>, XP_THREADS, xp_bytes<3, false, false>(), 1, d, ndesc, nplanes, bufs, st);
  return launch_xplane_k(k_xplane<2, 3, false, false>, XP_THREADS, xp_bytes<2, false, false>(), 1, d, ndesc, nplanes, bufs, st);
}

// block transforms with a real basis of at most 32 nodes (S at most 32 x 32): persistent k_xsmall
cudaError_t launch_xform_small(const GemmDesc* d_descs, int ndesc, int maxK, int64_t maxN, bool kcontig,
                               const Bufs& bufs, cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  if (maxK <= 16) return kcontig ? launch_xsmall_t<true, 16>(d_descs, ndesc, maxN, bufs, st)
                                 : launch_xsmall_t<false, 16>(d_descs, ndesc, maxN, bufs, st);
  if (maxK <= 32) return kcontig ? launch_xsmall_t<true, 32>(d_descs, ndesc, maxN, bufs, st)
                                 : launch_xsmall_t<false, 32>(d_descs, ndesc, maxN, bufs, st);
  return cudaErrorInvalidValue;
}

namespace {

// ---------------------------------------------------------------- complex S, 3 real products
// Complex eigenvector matrices (C blocks, global PML bases) with the 3-multiplication form
//   T1 = Sr Br, T2 = Si Bi, T3 = (Sr + Si)(Br + Bi);   Cr = T1 - T2,  Ci = T3 - T1 - T2
// 3 DMMA per complex 8x8x4 step instead of 4 (25% fewer tensor-pipe cycles; the sums are
// one DADD per fragment element).  CTA 64 x 64, 8 warps of 32 rows x 16 complex columns.
constexpr int X3_THREADS = 256;

template <bool KCONTIG>
__global__ void __launch_bounds__(X3_THREADS, 2) k_xform3m(const GemmDesc* __restrict__ descs, int gm, Bufs bufs) {
  extern __shared__ __align__(16) double xsm[];
  // the descriptor in shared memory: read from global memory it is re-fetched after every
  // barrier (the compiler cannot keep it in registers at the 128-register cap; ncu: ~10 % of
  // the stall samples were integer ops waiting on those loads)
  __shared__ GemmDesc sD;
  __shared__ int64_t sboff[4][X3_THREADS];  // KCONTIG: this thread's four B column offsets
  if (threadIdx.x < (int)(sizeof(GemmDesc) / 8))
    reinterpret_cast<int64_t*>(&sD)[threadIdx.x] = reinterpret_cast<const int64_t*>(descs + blockIdx.z)[threadIdx.x];
  __syncthreads();
  const GemmDesc& D = sD;
  const int M = D.M, K = D.K;
  const int64_t N2 = D.N2, N = (int64_t)D.N1 * D.N2;
  const int i0 = (int)(blockIdx.x % gm) * XT_M;  // row tiles fastest (B tile reuse in L2)
  const int64_t n0 = (int64_t)(blockIdx.x / gm) * XT_N;
  if (i0 >= M || n0 >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  const int g = lane >> 2, q = lane & 3;
  constexpr int STAGE = XSmem<false>::STAGE;
  const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off;
  const double2* A = reinterpret_cast<const double2*>(bufs.p[B_TAB]) + D.a_off;
  // A: 64 x 16 -> thread row tid/4, 4 consecutive j
  const int ai = tid >> 2, aj0 = (tid & 3) * 4;
  const bool arow_ok = (i0 + ai) < M;
  // KCONTIG: thread -> j = tid % 16, columns tid/16 + 16e (e < 4), their offsets in shared
  // memory (no registers to keep them in: this kernel is at the 128-register cap of two CTAs
  // per SM); otherwise thread -> column tid % 64, rows tid/64 + 4e
  int bj, bn0;
  int64_t bcol0, bn1_0, bn2_0;
  if (KCONTIG) {
    bj = tid & 15;
    bn0 = tid >> 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t n = n0 + bn0 + 16 * e;
      const int64_t n1 = n / N2, n2 = n - n1 * N2;
      sboff[e][tid] = n < N ? n1 * D.sB1 + n2 * D.sB2 : -1;
    }
  } else {
    bj = tid >> 6;
    bn0 = tid & 63;
  }
  {
    const int64_t n = n0 + bn0;
    bn1_0 = n / N2;
    bn2_0 = n - bn1_0 * N2;
    bcol0 = (n < N) ? bn1_0 * D.sB1 + bn2_0 * D.sB2 : -1;
  }
  auto load_chunk = [&](int stage, int j0) {
    double2* As = reinterpret_cast<double2*>(xsm + stage * STAGE);
    double2* Bs = As + XT_K * LDA_C;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + aj0 + e;
      const bool ok = arow_ok && j < K;
      cp_async16(As + (aj0 + e) * LDA_C + ai, ok ? A + (int64_t)(i0 + ai) * D.sAi + (int64_t)j * D.sAj : A, ok);
    }
    if (KCONTIG) {
      const int j = j0 + bj;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t o = sboff[e][tid];
        const bool ok = o >= 0 && j < K;
        cp_async16(Bs + bj * LDB_C + bn0 + 16 * e, ok ? B + o + j : B, ok);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = j0 + bj + 4 * e;
        const bool ok = bcol0 >= 0 && j < K;
        cp_async16(Bs + (bj + 4 * e) * LDB_C + bn0, ok ? B + bcol0 + (int64_t)j * D.sBj : B, ok);
      }
    }
  };
  double t1[4][2][2], t2[4][2][2], t3[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) t1[a][b][h] = t2[a][b][h] = t3[a][b][h] = 0.0;
  const int nchunks = (K + XT_K - 1) / XT_K;
  load_chunk(0, 0);
  cp_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) load_chunk((c + 1) & 1, (c + 1) * XT_K);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double2* As = reinterpret_cast<const double2*>(xsm + (c & 1) * STAGE);
    const double2* Bs = As + XT_K * LDA_C;
#pragma unroll
    for (int kk = 0; kk < XT_K; kk += 4) {
      double2 a[4], b[2];
      double sa[4], sb[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[(kk + q) * LDA_C + wm + 8 * i + g];
        sa[i] = a[i].x + a[i].y;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        b[j] = Bs[(kk + q) * LDB_C + wn + 8 * j + g];
        sb[j] = b[j].x + b[j].y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(t1[i][j][0], t1[i][j][1], a[i].x, b[j].x);
          dmma(t2[i][j][0], t2[i][j][1], a[i].y, b[j].y);
          dmma(t3[i][j][0], t3[i][j][1], sa[i], sb[j]);
        }
    }
    __syncthreads();
  }
  cp_wait<0>();
  double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off;
  // columns outer (wn + 8j + 2q + h, j < 2, h < 2; offsets stepped), rows inner
  {
    int64_t n = n0 + wn + 2 * q;
    int64_t n1 = n / N2, n2 = n - n1 * N2;
    const ColStep c1(1, N2), c7(7, N2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = e >> 1, h = e & 1;
      if (n < N) {
        const int64_t off = n1 * D.sC1 + n2 * D.sC2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i0 + wm + 8 * i + g;
          if (row >= M) continue;
          const double re = t1[i][j][h] - t2[i][j][h];
          const double im = t3[i][j][h] - t1[i][j][h] - t2[i][j][h];
          C[(int64_t)row * D.sCi + off] = make_double2(re, im);
        }
      }
      if (h) { n += 7; c7.advance(n1, n2, N2); }
      else { n += 1; c1.advance(n1, n2, N2); }
    }
  }
}

template <bool KCONTIG>
cudaError_t launch_3m(const GemmDesc* d, int ndesc, int maxM, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  const size_t sm = XSmem<false>::BYTES;
  cudaError_t e = cudaFuncSetAttribute(k_xform3m<KCONTIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  for (int z0 = 0; z0 < ndesc; z0 += 65535) {
    const int nzz = ndesc - z0 < 65535 ? ndesc - z0 : 65535;
    const int gm = (maxM + XT_M - 1) / XT_M;
    dim3 grid((unsigned)(((maxN + XT_N - 1) / XT_N) * gm), 1, (unsigned)nzz);
    k_xform3m<KCONTIG><<<grid, X3_THREADS, sm, st>>>(d + z0, gm, bufs);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_xform(const GemmDesc* d_descs, int ndesc, int maxM, int64_t maxN, bool real_s, bool kcontig,
                         const Bufs& bufs, cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  if (real_s) return kcontig ? launch_one<true, true>(d_descs, ndesc, maxM, maxN, bufs, st)
                             : launch_one<true, false>(d_descs, ndesc, maxM, maxN, bufs, st);
  return kcontig ? launch_3m<true>(d_descs, ndesc, maxM, maxN, bufs, st)
                 : launch_3m<false>(d_descs, ndesc, maxM, maxN, bufs, st);
}

}  // namespace lfds
