// Fast sine transforms for uniform blocks ("compute Fourier transforms in uniform parts via
// FFT").  For a block of n nodes with equal real steps h the eigenvectors are
//   W[p][c] = sqrt(2/(h N)) sin(pi (p+1)(c+1) / N),   N = n + 1          (natural mode order)
// so forward (F = W^T M = h W^T) and inverse (W) transforms are both a scaled DST-I:
//   C(c, col) = alpha * sum_{p=0}^{n-1} sin(pi (p+1)(c+1)/N) B(p, col),
//   alpha = sqrt(2h/N) (forward) or sqrt(2/(hN)) (inverse).
// DST-I via the odd extension y (length L = 2N: y_q = x_q, y_{L-q} = -x_q, y_0 = y_N = 0):
//   DFT_L(y)_k = -2i S(x)_k   =>   S(x)_k = (i/2) DFT_L(y)_k.
// The twiddles W_L^j = exp(-2 pi i j / L) come from the plan tables (GemmDesc.a_off).
// The length-L DFT uses the four-step split L = R1 * R2: R2 threads per column each run an
// R1-point FFT in registers, multiply by W_L^{n2 k1}, exchange through shared memory, then R1
// threads run R2-point FFTs.  Only the outputs k = 1..N-1 are kept.  FP64 CUDA-core
// arithmetic: ~5 L log2 L flops per column instead of the 4 n^2 of the dense real matrix.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <math_constants.h>
#include <stdint.h>

#include "lfds_internal.h"

namespace lfds {
namespace {

namespace cg = cooperative_groups;

// cluster barrier without release semantics: orders only execution (used where the CTAs just
// need each other's reads of their own shared memory done — a release would also wait for all
// of this thread's outstanding global stores)
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}

struct zc2 {
  double x, y;
};
__device__ __forceinline__ zc2 zadd(zc2 a, zc2 b) { return zc2{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ zc2 zsub(zc2 a, zc2 b) { return zc2{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ zc2 zmul(zc2 a, zc2 b) {
  return zc2{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}

// in-register radix-2 DIT FFT (forward, e^{-2 pi i k n / R}); all indices compile-time.
// Twiddles W_len^j = W_L^{j L/len}: the trivial ones are applied without a general complex
// multiply (W^0 = 1, W^{len/4} = -i, W^{len/8} = (1-i)/sqrt2, W^{3len/8} = -(1+i)/sqrt2 — in a
// 16-point FFT only 4 of the 32 butterflies need one); the others are warp-uniform broadcast
// reads of the W_L table.
template <int LEN, int J, int L>
__device__ __forceinline__ zc2 twiddle_mul(zc2 b, const double2* __restrict__ twl) {
  constexpr double SH = 0.70710678118654752440;  // sqrt(1/2)
  if constexpr (J == 0) {
    return b;
  } else if constexpr (4 * J == LEN) {
    return zc2{b.y, -b.x};
  } else if constexpr (8 * J == LEN) {
    return zc2{SH * (b.x + b.y), SH * (b.y - b.x)};
  } else if constexpr (8 * J == 3 * LEN) {
    return zc2{SH * (b.y - b.x), -SH * (b.x + b.y)};
  } else {
    const double2 w2 = twl[J * (L / LEN)];
    return zmul(zc2{w2.x, w2.y}, b);
  }
}

template <int R, int L, int LEN, int J>
__device__ __forceinline__ void fft_butterflies(zc2 (&v)[R], const double2* __restrict__ twl) {
  if constexpr (J < LEN / 2) {
#pragma unroll
    for (int i = 0; i < R; i += LEN) {
      const zc2 u = v[i + J], t = twiddle_mul<LEN, J, L>(v[i + J + LEN / 2], twl);
      v[i + J] = zadd(u, t);
      v[i + J + LEN / 2] = zsub(u, t);
    }
    fft_butterflies<R, L, LEN, J + 1>(v, twl);
  }
}

template <int R, int L, int LEN>
__device__ __forceinline__ void fft_stages(zc2 (&v)[R], const double2* __restrict__ twl) {
  if constexpr (LEN <= R) {
    fft_butterflies<R, L, LEN, 0>(v, twl);
    fft_stages<R, L, 2 * LEN>(v, twl);
  }
}

template <int R, int L>
__device__ __forceinline__ void fft_reg(zc2 (&v)[R], const double2* __restrict__ twl) {
  // bit reversal
#pragma unroll
  for (int i = 0; i < R; ++i) {
    int j = 0;
#pragma unroll
    for (int b = 1, t = i; b < R; b <<= 1, t >>= 1) j = (j << 1) | (t & 1);
    if (j > i) {
      zc2 t2 = v[i];
      v[i] = v[j];
      v[j] = t2;
    }
  }
  fft_stages<R, L, 2>(v, twl);
}

// Mixed-radix in-register DFT of length R = 2^a 3^b 5^c (compile-time Cooley-Tukey, decimation
// in time: R = P Q with P the smallest prime factor; X[k1 + P k2] = sum_n2 W_Q^{n2 k2}
// W_R^{n2 k1} sum_n1 W_P^{n1 k1} x[Q n1 + n2]); twiddles from the W_L table (R divides L).
template <int P>
__device__ __forceinline__ void dft_small(zc2 (&x)[P]) {
  if constexpr (P == 2) {
    const zc2 a = x[0], b = x[1];
    x[0] = zadd(a, b);
    x[1] = zsub(a, b);
  } else if constexpr (P == 3) {  // W = e^{-2 pi i/3}
    constexpr double h = 0.86602540378443864676;  // sqrt(3)/2
    const zc2 a = x[0], t1 = zadd(x[1], x[2]), d = zsub(x[1], x[2]);
    const zc2 t2{a.x - 0.5 * t1.x, a.y - 0.5 * t1.y};
    x[0] = zadd(a, t1);
    x[1] = zc2{t2.x + h * d.y, t2.y - h * d.x};  // t2 - i h d
    x[2] = zc2{t2.x - h * d.y, t2.y + h * d.x};  // t2 + i h d
  } else {  // P == 5, W = e^{-2 pi i/5}
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
    const zc2 a = x[0];
    const zc2 t1 = zadd(x[1], x[4]), t2 = zadd(x[2], x[3]), t3 = zsub(x[1], x[4]), t4 = zsub(x[2], x[3]);
    const zc2 r1{a.x + c1 * t1.x + c2 * t2.x, a.y + c1 * t1.y + c2 * t2.y};
    const zc2 r2{a.x + c2 * t1.x + c1 * t2.x, a.y + c2 * t1.y + c1 * t2.y};
    const zc2 i1{s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y};
    const zc2 i2{s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y};
    x[0] = zc2{a.x + t1.x + t2.x, a.y + t1.y + t2.y};
    x[1] = zc2{r1.x + i1.y, r1.y - i1.x};  // r1 - i i1
    x[4] = zc2{r1.x - i1.y, r1.y + i1.x};
    x[2] = zc2{r2.x + i2.y, r2.y - i2.x};
    x[3] = zc2{r2.x - i2.y, r2.y + i2.x};
  }
}

template <int R, int L>
__device__ __forceinline__ void dft_reg(zc2 (&v)[R], const double2* __restrict__ twl) {
  if constexpr ((R & (R - 1)) == 0) {
    fft_reg<R, L>(v, twl);
  } else if constexpr (R == 3 || R == 5) {
    dft_small<R>(v);
  } else {
    constexpr int P = R % 2 == 0 ? 2 : R % 3 == 0 ? 3 : 5, Q = R / P;
    zc2 A[P][Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) {
      zc2 x[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) x[n1] = v[Q * n1 + n2];
      dft_small<P>(x);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) {
        if (n2 * k1 == 0) {
          A[k1][n2] = x[k1];
        } else {
          const double2 w = twl[(n2 * k1 * (L / R)) % L];
          A[k1][n2] = zmul(x[k1], zc2{w.x, w.y});
        }
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      dft_reg<Q, L>(A[k1], twl);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) v[k1 + P * k2] = A[k1][k2];
    }
  }
}

constexpr int DST_THREADS = 128;  // 8 columns per CTA at L = 256: small CTAs, many resident per SM

__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0));
}

template <int R1, int R2, bool KCONTIG>
__global__ void __launch_bounds__(DST_THREADS, (R1 <= 16 && R2 <= 16) ? 5 : R1 == 20 ? 4 : 1) k_dst(const GemmDesc* __restrict__ descs, Bufs bufs) {
  constexpr int L = R1 * R2, N = L / 2;
  constexpr int CPB = DST_THREADS / R2;      // columns per CTA
  constexpr int LDT = CPB + 1;               // tile row stride (complex)
  extern __shared__ __align__(16) double2 dsm[];
  // buffer: tile [N-1][LDT] (load, later output staging) aliased with exchange [R1][R2][CPB]
  double2* tile = dsm;
  double2* ex = dsm;
  __shared__ double2 twl[L];                 // W_L^j, j < L
  __shared__ int64_t colB[CPB], colC[CPB];
  const GemmDesc& D = descs[blockIdx.z];
  const int n = N - 1;
  const int64_t N2 = D.N2, NC = (int64_t)D.N1 * D.N2;
  const int64_t c0 = (int64_t)blockIdx.x * CPB;
  if (c0 >= NC) return;
  const int tid = threadIdx.x;
  for (int j = tid; j < L; j += DST_THREADS) twl[j] = __ldg(reinterpret_cast<const double2*>(bufs.p[B_TAB]) + D.a_off + j);
  if (tid < CPB) {
    const int64_t col = c0 + tid;
    const int64_t n1 = col / N2, n2 = col - n1 * N2;
    colB[tid] = col < NC ? D.b_off + n1 * D.sB1 + n2 * D.sB2 : -1;
    colC[tid] = col < NC ? D.c_off + n1 * D.sC1 + n2 * D.sC2 : -1;
  }
  __syncthreads();
  const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]);
  double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]);
  // ---- load the CPB columns (n values each) into tile[p][col]: every copy is an async
  // 16-byte cp.async, so all of a thread's loads are in flight at once
  if (KCONTIG) {  // a column is contiguous in memory: sweep along p
    for (int idx = tid; idx < n * CPB; idx += DST_THREADS) {
      const int col = idx / n, p = idx - col * n;
      const int64_t b = colB[col];
      cp_async16z(&tile[p * LDT + col], b >= 0 ? B + b + p : B, b >= 0);
    }
  } else {        // consecutive columns are adjacent in memory: sweep along col
    for (int idx = tid; idx < n * CPB; idx += DST_THREADS) {
      const int p = idx / CPB, col = idx - p * CPB;
      const int64_t b = colB[col];
      cp_async16z(&tile[p * LDT + col], b >= 0 ? B + b + (int64_t)p * D.sBj : B, b >= 0);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  // thread -> (column, FFT lane t): the CPB columns of a warp are adjacent, so a warp's
  // accesses at fixed t cover whole 128-byte rows, and its twiddles W_L^{t k1} are shared by
  // the CPB lanes of each t (shared-memory broadcast)
  const int col = tid % CPB, t = tid / CPB;
  // ---- step 1: thread n2 = t: R1-point FFT over n1 of y[R2 n1 + n2], twiddle W_L^{n2 k1}
  zc2 a[R1];
#pragma unroll
  for (int n1 = 0; n1 < R1; ++n1) {
    const int q = R2 * n1 + t;
    zc2 v{0, 0};
    if (q > 0 && q < N) {
      const double2 w = tile[(q - 1) * LDT + col];
      v = zc2{w.x, w.y};
    } else if (q > N) {
      const double2 w = tile[(L - q - 1) * LDT + col];
      v = zc2{-w.x, -w.y};
    }
    a[n1] = v;
  }
  dft_reg<R1, L>(a, twl);
#pragma unroll
  for (int k1 = 1; k1 < R1; ++k1) {
    const double2 w = twl[(t * k1) % L];
    a[k1] = zmul(a[k1], zc2{w.x, w.y});
  }
  __syncthreads();  // tile fully consumed
  // exchange [k1][n2][col]: conflict-free writes (fixed k1) and reads (fixed n2)
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) ex[(k1 * R2 + t) * CPB + col] = make_double2(a[k1].x, a[k1].y);
  __syncthreads();
  // ---- step 3: rows k1 = t, t + R2, ...: R2-point FFT over n2 -> Y[k1 + R1 k2], keep k < N.
  constexpr int RPT = (R1 + R2 - 1) / R2;  // rows per thread
  zc2 b[RPT][R2];
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const int k1 = t + rr * R2;
    if (k1 < R1) {
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) {
        const double2 w = ex[(k1 * R2 + n2) * CPB + col];
        b[rr][n2] = zc2{w.x, w.y};
      }
      fft_reg<R2, L>(b[rr], twl);
    }
  }
  const double half = 0.5 * D.scale;
  if (D.sCi != 1) {  // strided output rows: store straight from registers (a warp writes whole rows)
    const int64_t o = colC[col];
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) {
      const int k1 = t + rr * R2;
      if (k1 < R1 && o >= 0) {
#pragma unroll
        for (int k2 = 0; k2 < R2 / 2; ++k2) {
          const int k = k1 + R1 * k2;
          if (k >= 1 && k < N) C[o + (int64_t)(k - 1) * D.sCi] = make_double2(-half * b[rr][k2].y, half * b[rr][k2].x);
        }
      }
    }
    return;
  }
  __syncthreads();  // exchange consumed; reuse as output tile[c][col]
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const int k1 = t + rr * R2;
    if (k1 < R1) {
#pragma unroll
      for (int k2 = 0; k2 < R2 / 2; ++k2) {
        const int k = k1 + R1 * k2;
        if (k >= 1 && k < N) tile[(k - 1) * LDT + col] = make_double2(-half * b[rr][k2].y, half * b[rr][k2].x);
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < n * CPB; idx += DST_THREADS) {  // output column contiguous
    const int cc = idx / n, c = idx - cc * n;
    const int64_t o = colC[cc];
    if (o >= 0) C[o + c] = tile[c * LDT + cc];
  }
}

template <int R1, int R2, bool KC>
cudaError_t dst_launch(const GemmDesc* d, int ndesc, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  constexpr int L = R1 * R2, N = L / 2, CPB = DST_THREADS / R2;
  const size_t tile = (size_t)(N - 1) * (CPB + 1) * sizeof(double2);
  const size_t ex = (size_t)CPB * R1 * R2 * sizeof(double2);
  const size_t sm = tile > ex ? tile : ex;
  cudaError_t e = cudaFuncSetAttribute(k_dst<R1, R2, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  for (int z0 = 0; z0 < ndesc; z0 += 65535) {
    const int nzz = ndesc - z0 < 65535 ? ndesc - z0 : 65535;
    dim3 grid((unsigned)((maxN + CPB - 1) / CPB), 1, (unsigned)nzz);
    k_dst<R1, R2, KC><<<grid, DST_THREADS, sm, st>>>(d + z0, bufs);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- TMA-fed strided variant
// k_dst for strided columns (y direction) with its tiles moved by the tensor memory
// accelerator: per descriptor a 3-D tensor map (2 N2 doubles x K rows x N1 planes, the box one
// 8-column tile of all K rows of one plane), one cp.async.bulk.tensor per tile completing on an
// mbarrier, NBUF tiles in flight per CTA in a persistent loop over the (descriptor, plane,
// column-tile) items.  k_dst issues 8 cp.async per thread per tile and its five CTAs per SM
// meet at their wait_all; here one thread issues one instruction per tile and the FFTs of a
// tile overlap the copies of the next ones.  Same arithmetic and output order as k_dst.
__device__ __forceinline__ uint32_t dsmem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R1, int R2, int NBUF>
__global__ void __launch_bounds__(DST_THREADS, (R1 <= 16 && R2 <= 16) ? 3 : 1) k_dstt(
    const GemmDesc* __restrict__ descs, const CUtensorMap* __restrict__ maps, int ndesc, int col_tiles,
    int tiles_per_desc, Bufs bufs) {
  constexpr int L = R1 * R2, N = L / 2, n = N - 1;
  constexpr int CPB = DST_THREADS / R2;
  constexpr int TILE = n * CPB;                  // dense box [p][col] (a multiple of 128 B)
  extern __shared__ __align__(16) double2 dsmt[];
  // tensor-copy destinations must be 128-B aligned: the launch adds 128 B of slack
  double2* tiles = reinterpret_cast<double2*>(((uintptr_t)dsmt + 127) & ~(uintptr_t)127);  // [NBUF][TILE]
  double2* ex = tiles + NBUF * TILE;             // [R1][R2][CPB]
  __shared__ double2 twl[L];
  __shared__ __align__(8) uint64_t full[NBUF];
  const int tid = threadIdx.x;
  const int64_t items = (int64_t)ndesc * tiles_per_desc;
  if ((int64_t)blockIdx.x >= items) return;
  {
    const GemmDesc& D0 = descs[0];
    for (int j = tid; j < L; j += DST_THREADS) twl[j] = __ldg(reinterpret_cast<const double2*>(bufs.p[B_TAB]) + D0.a_off + j);
  }
  if (tid == 0) {
    for (int q = 0; q < NBUF; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(dsmem_addr(&full[q])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t it, int bf) {
    if (tid != 0 || it >= items) return;
    const int d = (int)(it / tiles_per_desc), t = (int)(it % tiles_per_desc);
    const int plane = t / col_tiles, c0 = (t % col_tiles) * CPB;
    const CUtensorMap* m = maps + d;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(dsmem_addr(&full[bf])),
                 "r"((uint32_t)(TILE * 16))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            dsmem_addr(tiles + bf * TILE)),
        "l"(m), "r"(2 * c0), "r"(0), "r"(plane), "r"(dsmem_addr(&full[bf]))
        : "memory");
  };
  const int64_t G = gridDim.x;
#pragma unroll
  for (int q = 0; q < NBUF - 1; ++q) issue(blockIdx.x + q * G, q);
  const int col = tid % CPB, t = tid / CPB;
  int k = 0;
  for (int64_t it = blockIdx.x; it < items; it += G, ++k) {
    const int bf = k % NBUF;
    __syncthreads();  // buffer (k - 1) % NBUF and the exchange of tile k - 1 fully consumed
    issue(it + (NBUF - 1) * G, (k + NBUF - 1) % NBUF);
    {
      const uint32_t bar = dsmem_addr(&full[bf]), par = (uint32_t)((k / NBUF) & 1);
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
          "r"(par)
          : "memory");
    }
    const int d = (int)(it / tiles_per_desc), ti = (int)(it % tiles_per_desc);
    const GemmDesc& D = descs[d];
    const int plane = ti / col_tiles, c0 = (ti % col_tiles) * CPB;
    const double2* tile = tiles + bf * TILE;
    zc2 a[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int q = R2 * n1 + t;
      zc2 v{0, 0};
      if (q > 0 && q < N) {
        const double2 w = tile[(q - 1) * CPB + col];
        v = zc2{w.x, w.y};
      } else if (q > N) {
        const double2 w = tile[(L - q - 1) * CPB + col];
        v = zc2{-w.x, -w.y};
      }
      a[n1] = v;
    }
    dft_reg<R1, L>(a, twl);
#pragma unroll
    for (int k1 = 1; k1 < R1; ++k1) {
      const double2 w = twl[(t * k1) % L];
      a[k1] = zmul(a[k1], zc2{w.x, w.y});
    }
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) ex[(k1 * R2 + t) * CPB + col] = make_double2(a[k1].x, a[k1].y);
    __syncthreads();
    constexpr int RPT = (R1 + R2 - 1) / R2;
    zc2 b[RPT][R2];
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) {
      const int k1 = t + rr * R2;
      if (k1 < R1) {
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
          const double2 w = ex[(k1 * R2 + n2) * CPB + col];
          b[rr][n2] = zc2{w.x, w.y};
        }
        fft_reg<R2, L>(b[rr], twl);
      }
    }
    const double half = 0.5 * D.scale;
    double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]);
    const int64_t n2c = c0 + col;
    if (n2c < D.N2) {  // strided output rows, straight from registers (a warp writes whole rows)
      const int64_t o = D.c_off + (int64_t)plane * D.sC1 + n2c * D.sC2;
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int k1 = t + rr * R2;
        if (k1 < R1) {
#pragma unroll
          for (int k2 = 0; k2 < R2 / 2; ++k2) {
            const int kk = k1 + R1 * k2;
            if (kk >= 1 && kk < N) C[o + (int64_t)(kk - 1) * D.sCi] = make_double2(-half * b[rr][k2].y, half * b[rr][k2].x);
          }
        }
      }
    }
  }
}

// driver entry point of cuTensorMapEncodeTiled (the runtime links no libcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <int R1, int R2>
cudaError_t dstt_launch(const GemmDesc* d, const void* maps, int ndesc, int maxN2, int maxN1, const Bufs& bufs,
                        cudaStream_t st) {
  constexpr int L = R1 * R2, N = L / 2, n = N - 1, CPB = DST_THREADS / R2, NBUF = 2;
  const size_t sm = (size_t)(NBUF * n * CPB + CPB * R1 * R2) * sizeof(double2) + 128;
  auto kern = k_dstt<R1, R2, NBUF>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, DST_THREADS, sm)) != cudaSuccess) return e;
  const int col_tiles = (maxN2 + CPB - 1) / CPB;
  const int tiles_per_desc = col_tiles * maxN1;
  const int64_t items = (int64_t)ndesc * tiles_per_desc;
  const int64_t grid = std::min<int64_t>(items, (int64_t)std::max(1, per) * sms);
  kern<<<(unsigned)grid, DST_THREADS, sm, st>>>(d, reinterpret_cast<const CUtensorMap*>(maps), ndesc, col_tiles,
                                                tiles_per_desc, bufs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- warp-autonomous variant
// A warp transforms CPW = 32/R2 columns at a time, R2 lanes per column, with no CTA barrier:
// lane t of a column loads its R1 inputs y[R2 n1 + t] of the odd extension straight from
// global memory into registers (for contiguous columns one load instruction covers R2
// consecutive elements; for adjacent strided columns the CPW columns of a warp are adjacent
// in memory, so every 32-byte sector is used), runs the first R1-point FFTs, exchanges
// through a per-warp shared-memory transpose (__syncwarp only), runs the R2-point FFTs and
// stores its outputs directly.  Many independent warps keep many loads in flight; each warp
// walks its columns in a grid-stride loop.  Used for contiguous columns (x direction): for
// strided columns two adjacent columns per warp use only 32-byte pieces of each row, and the
// CTA-tiled k_dst (8 adjacent columns per row) is faster there.
template <int R1>
struct DstwWarps {  // warps per CTA (static shared memory: per-warp exchange + two twiddle tables)
  static constexpr int value = R1 > 16 ? 2 : 4;
};

template <int R1, int R2>
__global__ void __launch_bounds__(DstwWarps<R1>::value * 32) k_dstw(const GemmDesc* __restrict__ descs, int ndesc, int64_t maxN,
                                                          Bufs bufs) {
  constexpr int L = R1 * R2, N = L / 2, CPW = 32 / R2, LDE = R2 + 1, DSTW_WARPS = DstwWarps<R1>::value;
  __shared__ double2 twl[L];
  __shared__ double2 tws[R1 * R2];                       // W_L^{t k1} at [k1][t]
  __shared__ double2 exs[DSTW_WARPS][CPW * R1 * LDE];    // per-warp exchange
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cw = lane / R2, t = lane % R2;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* TW = TAB + descs[0].a_off;              // one length per launch
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    twl[j] = __ldg(TW + j);
    tws[j] = __ldg(TW + ((j % R2) * (j / R2)) % L);
  }
  __syncthreads();
  double2* ex = exs[warp];
  const int64_t groups_per_desc = (maxN + CPW - 1) / CPW;
  const int64_t total = groups_per_desc * ndesc;
  for (int64_t gi = (int64_t)blockIdx.x * DSTW_WARPS + warp; gi < total; gi += (int64_t)gridDim.x * DSTW_WARPS) {
    const GemmDesc& D = descs[gi / groups_per_desc];
    const int64_t col = (gi % groups_per_desc) * CPW + cw, NC = (int64_t)D.N1 * D.N2;
    const bool ok = col < NC;
    const int64_t n1c = ok ? col / D.N2 : 0, n2c = ok ? col - n1c * D.N2 : 0;
    const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off + n1c * D.sB1 + n2c * D.sB2;
    double2* C = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off + n1c * D.sC1 + n2c * D.sC2;
    const int64_t sb = D.sBj, sc = D.sCi;
    // ---- loads: y[q], q = R2 n1 + t (x_{q-1} for 0 < q < N, -x_{L-q-1} for q > N, 0 at 0, N)
    zc2 a[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int q = R2 * n1 + t;
      zc2 v{0, 0};
      if (ok && q > 0 && q < N) {
        const double2 w = __ldg(B + (int64_t)(q - 1) * sb);
        v = zc2{w.x, w.y};
      } else if (ok && q > N) {
        const double2 w = __ldg(B + (int64_t)(L - q - 1) * sb);
        v = zc2{-w.x, -w.y};
      }
      a[n1] = v;
    }
    dft_reg<R1, L>(a, twl);
#pragma unroll
    for (int k1 = 1; k1 < R1; ++k1) {
      const double2 w = tws[k1 * R2 + t];
      a[k1] = zmul(a[k1], zc2{w.x, w.y});
    }
    __syncwarp();  // previous column group's exchange reads are done
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) ex[(cw * R1 + k1) * LDE + t] = make_double2(a[k1].x, a[k1].y);
    __syncwarp();
    // ---- R2-point FFTs: lane t of the column takes rows k1 = t, t + R2, ...; outputs k = k1 + R1 k2
#pragma unroll
    for (int rr = 0; rr < (R1 + R2 - 1) / R2; ++rr) {
      const int k1 = t + rr * R2;
      if (k1 < R1) {
        zc2 b[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
          const double2 w = ex[(cw * R1 + k1) * LDE + n2];
          b[n2] = zc2{w.x, w.y};
        }
        fft_reg<R2, L>(b, twl);
        const double half = 0.5 * D.scale;
#pragma unroll
        for (int k2 = 0; k2 < R2 / 2; ++k2) {
          const int k = k1 + R1 * k2;
          if (ok && k >= 1 && k < N) C[(int64_t)(k - 1) * sc] = make_double2(-half * b[k2].y, half * b[k2].x);
        }
      }
    }
  }
}

template <int R1, int R2>
cudaError_t dstw_launch(const GemmDesc* d, int ndesc, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  constexpr int DSTW_WARPS = DstwWarps<R1>::value;
  int per_sm = 0, dev = 0, sms = 148;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dstw<R1, R2>, DSTW_WARPS * 32, 0);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int CPW = 32 / R2;
  const int64_t warps = ((maxN + CPW - 1) / CPW) * ndesc;
  const int64_t grid = std::min<int64_t>((warps + DSTW_WARPS - 1) / DSTW_WARPS, (int64_t)sms * std::max(1, per_sm));
  k_dstw<R1, R2><<<(unsigned)grid, DSTW_WARPS * 32, 0, st>>>(d, ndesc, maxN, bufs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- plane (2-D) transform
// A uniform x uniform block with n nodes on both axes: the tensor-product transform
// C = a_y a_x S_y B S_x^T of every (r, k) plane in ONE pass over the block (the separate x and
// y passes read and write the volume twice).  The plane lives in shared memory between the two
// 1-D transforms: one CTA holds it for n <= 31 (15 KB), a cluster of CL = ceil(n/32) CTAs for
// larger n (n = 63: 2 CTAs of 33 KB), CTA q owning the x-modes [q RPC, (q+1) RPC) of all rows:
//   x phase: CTA q transforms the rows [q RPC, (q+1) RPC) exactly like k_dstw (loads straight
//            from global memory into registers, per-warp exchange) and stores every output
//            (row, x-mode l) into the shared memory of the CTA owning l (DSMEM stores);
//   cluster barrier (release / acquire);
//   y phase: CTA q transforms its RPC columns from local shared memory and stores them (two
//            adjacent columns per warp instruction: whole 32-byte sectors).
// Clusters stride over the (block, plane) items; a second cluster barrier ends each item.  Used
// for L = 2(n+1) in {32, 64, 128}; see dst2_supported() for why not beyond.
template <int R1, int R2>
struct Dst2Cfg {
  static constexpr int L = R1 * R2, N = L / 2, n = N - 1;
  static constexpr int CL = (n + 31) / 32;                  // CTAs per cluster (<= 8)
  static constexpr int RPC = (n + CL - 1) / CL;              // x-modes / rows per CTA
  static constexpr int LDT = RPC % 2 ? RPC : RPC + 1;        // odd: conflict-free column reads
  static constexpr int WARPS = R1 > 16 ? 2 : 4, CPW = 32 / R2, LDE = R2 + 1;
  static constexpr size_t smem = (size_t)n * LDT * sizeof(double2);
};

template <int R1, int R2>
__device__ __forceinline__ void dst2_fft(zc2 (&a)[R1], const double2* twl, const double2* tws, double2* ex, int cw,
                                         int t, zc2 (&b)[(R1 + R2 - 1) / R2][R2]) {
  constexpr int L = R1 * R2, LDE = R2 + 1;
  dft_reg<R1, L>(a, twl);
#pragma unroll
  for (int k1 = 1; k1 < R1; ++k1) {
    const double2 w = tws[k1 * R2 + t];
    a[k1] = zmul(a[k1], zc2{w.x, w.y});
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) ex[(cw * R1 + k1) * LDE + t] = make_double2(a[k1].x, a[k1].y);
  __syncwarp();
#pragma unroll
  for (int rr = 0; rr < (R1 + R2 - 1) / R2; ++rr) {
    const int k1 = t + rr * R2;
    if (k1 < R1) {
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) {
        const double2 w = ex[(cw * R1 + k1) * LDE + n2];
        b[rr][n2] = zc2{w.x, w.y};
      }
      fft_reg<R2, L>(b[rr], twl);
    }
  }
}

template <int R1, int R2>
__global__ void __launch_bounds__(Dst2Cfg<R1, R2>::WARPS * 32) k_dst2(const Dst2Desc* __restrict__ descs, int ndesc,
                                                                      int nplanes, Bufs bufs) {
  using C = Dst2Cfg<R1, R2>;
  constexpr int L = C::L, N = C::N, n = C::n, RPC = C::RPC, LDT = C::LDT, CPW = C::CPW, RPT = (R1 + R2 - 1) / R2;
  extern __shared__ __align__(16) double2 Tsm[];   // [row q < n][x-mode l - q0 < RPC], row stride LDT
  __shared__ double2 twl[L];
  __shared__ double2 tws[R1 * R2];                  // W_L^{t k1} at [k1][t]
  __shared__ double2 exs[C::WARPS][CPW * R1 * C::LDE];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cw = lane / R2, t = lane % R2;
  {  // one length per launch: every descriptor has the same twiddle table
    const double2* TW = reinterpret_cast<const double2*>(bufs.p[B_TAB]) + descs[0].tw_off;
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
      twl[j] = __ldg(TW + j);
      tws[j] = __ldg(TW + ((j % R2) * (j / R2)) % L);
    }
  }
  __syncthreads();
  double2* ex = exs[warp];
  const int r0 = q * RPC, nr = min(RPC, n - r0);
  // persistent clusters: work item w = (descriptor, plane), clusters stride over the items
  const int64_t total = (int64_t)ndesc * nplanes, ncl = gridDim.x / C::CL;
  auto load_row = [&](const double2* B, int64_t sBr, int g, zc2 (&a)[R1]) {
    const int rl = g * CPW + cw;
    const bool ok = rl < nr;
    const double2* Br = B + (int64_t)(ok ? r0 + rl : 0) * sBr;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int qq = R2 * n1 + t;
      zc2 v{0, 0};
      if (ok && qq > 0 && qq < N) {
        const double2 w = __ldg(Br + (qq - 1));
        v = zc2{w.x, w.y};
      } else if (ok && qq > N) {
        const double2 w = __ldg(Br + (L - qq - 1));
        v = zc2{-w.x, -w.y};
      }
      a[n1] = v;
    }
  };
  for (int64_t w = blockIdx.x / C::CL; w < total; w += ncl) {
    const Dst2Desc& D = descs[w / nplanes];
    const int64_t plane = w % nplanes;
    const double2* B = reinterpret_cast<const double2*>(bufs.p[D.b_buf]) + D.b_off + plane * D.sB1;
    double2* Cg = reinterpret_cast<double2*>(bufs.p[D.c_buf]) + D.c_off + plane * D.sC1;
    // ---- x phase: rows r0 .. r0+nr-1, CPW rows per warp step, outputs to the owner's Tsm
    const double hx = 0.5 * D.ax;
    for (int g = warp; g * CPW < nr; g += C::WARPS) {
      const int rl = g * CPW + cw, r = r0 + rl;
      const bool ok = rl < nr;
      zc2 a[R1];
      load_row(B, D.sBr, g, a);
      zc2 b[RPT][R2];
      dst2_fft<R1, R2>(a, twl, tws, ex, cw, t, b);
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int k1 = t + rr * R2;
        if (k1 < R1 && ok) {
#pragma unroll
          for (int k2 = 0; k2 < R2 / 2; ++k2) {
            const int k = k1 + R1 * k2;
            if (k >= 1 && k < N) {
              const int l = k - 1, o = l / RPC;
              double2* dst = C::CL == 1 ? Tsm : cluster.map_shared_rank(Tsm, o);
              dst[r * LDT + (l - o * RPC)] = make_double2(-hx * b[rr][k2].y, hx * b[rr][k2].x);
            }
          }
        }
      }
    }
    // the plane's x-transformed rows are complete in the cluster (one CTA: a block barrier)
    if constexpr (C::CL == 1) __syncthreads(); else cluster.sync();
    // ---- y phase: columns (x-modes) r0 .. r0+nr-1 of all n rows, CPW columns per warp step
    const double hy = 0.5 * D.ay;
    const bool rows_out = D.sCr != n;  // (uniform over the cluster: one descriptor per item)
    for (int g = warp; g * CPW < nr; g += C::WARPS) {
      const int cl = g * CPW + cw;
      const bool ok = cl < nr;
      const int cc = ok ? cl : 0;
      zc2 a[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int qq = R2 * n1 + t;
        zc2 v{0, 0};
        if (qq > 0 && qq < N) {
          const double2 x = Tsm[(qq - 1) * LDT + cc];
          v = zc2{x.x, x.y};
        } else if (qq > N) {
          const double2 x = Tsm[(L - qq - 1) * LDT + cc];
          v = zc2{-x.x, -x.y};
        }
        a[n1] = v;
      }
      zc2 b[RPT][R2];
      dst2_fft<R1, R2>(a, twl, tws, ex, cw, t, b);
      // output rows strided in a larger array (step 7: u rows of the global grid): back into the
      // column in place (this warp read all of it above) and stored as whole rows below; a
      // contiguous output plane (step 1: the block's mode space) takes the direct stores
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int k1 = t + rr * R2;
        if (k1 < R1 && ok) {
#pragma unroll
          for (int k2 = 0; k2 < R2 / 2; ++k2) {
            const int k = k1 + R1 * k2;
            if (k >= 1 && k < N) {
              const double2 v = make_double2(-hy * b[rr][k2].y, hy * b[rr][k2].x);
              if (rows_out) Tsm[(k - 1) * LDT + cl] = v;
              else Cg[(int64_t)(k - 1) * D.sCr + r0 + cl] = v;
            }
          }
        }
      }
    }
    if (rows_out) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < n * nr; idx += blockDim.x) {  // row m: x-modes r0 .. r0+nr-1
        const int m = idx / nr, c = idx - m * nr;
        Cg[(int64_t)m * D.sCr + r0 + c] = Tsm[m * LDT + c];
      }
    }
    // every CTA has read its Tsm before the next x phase writes into it; with rows_out the CTA
    // also WROTE its Tsm above, and the peer's next remote stores must be ordered after those
    // local writes: a release/acquire cluster barrier (a relaxed arrive only orders the reads)
    if constexpr (C::CL == 1) __syncthreads();
    else if (rows_out) cluster.sync();
    else cluster_sync_relaxed();
  }
}

template <int R1, int R2>
cudaError_t dst2_launch(const Dst2Desc* d, int ndesc, int nplanes, const Bufs& bufs, cudaStream_t st) {
  using C = Dst2Cfg<R1, R2>;
  auto kern = k_dst2<R1, R2>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(C::WARPS * 32, 1, 1);
  cfg.dynamicSmemBytes = C::smem;
  cfg.stream = st;
  // clusters stride over the (descriptor, plane) items: 4 x the co-resident clusters (measured
  // better than exactly one wave: a cluster that finishes early is replaced at once; loading
  // the next item's rows ahead into registers measured slower at L = 64 / 128)
  cfg.gridDim = dim3(C::CL, 1, 1);
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (e != cudaSuccess) return e;
  const int64_t items = (int64_t)ndesc * nplanes;
  ncl = (int)std::min<int64_t>(std::max(1, ncl) * 4LL, items);
  cfg.gridDim = dim3((unsigned)(ncl * C::CL), 1, 1);
  e = cudaLaunchKernelEx(&cfg, kern, d, ndesc, nplanes, bufs);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

bool dst2_supported(int n) {
  // lengths where the plane transform beats the x pass + y pass (tools/plane_dst_ab.py on the
  // C4 grid: L = 64 7.97 -> 6.98 ms, L = 128 8.04 -> 7.52 ms per step of sine stages).  At
  // L = 256 (4-CTA clusters) and 320 (5) a plane needs 2 or 1 CTAs per SM (shared memory
  // 110 / 138 KB, ~220 registers per thread): too few warps to hide the load latency
  // (L = 256: 5.99 -> 6.64 ms, L = 320: 6.41 -> 14.7 ms), so those stay on the 1-D passes.
  const int L = 2 * (n + 1);
  return L == 32 || L == 64 || L == 128;
}

cudaError_t launch_dst2(const Dst2Desc* d_descs, int ndesc, int n, int nplanes, const Bufs& bufs, cudaStream_t st) {
  if (ndesc <= 0 || nplanes <= 0) return cudaSuccess;
  switch (2 * (n + 1)) {
    case 32: return dst2_launch<4, 8>(d_descs, ndesc, nplanes, bufs, st);
    case 64: return dst2_launch<8, 8>(d_descs, ndesc, nplanes, bufs, st);
    case 128: return dst2_launch<8, 16>(d_descs, ndesc, nplanes, bufs, st);
    default: return cudaErrorInvalidValue;
  }
}

bool dst_supported(int n) {
  const int L = 2 * (n + 1);
  if (L == 16 || L == 32 || L == 64 || L == 128 || L == 256 || L == 512) return true;
  // mixed radix: L = R1 * 16 with R1 in {3, 5, 6, 10, 12, 20} (e.g. n = 159: L = 320)
  const int r1 = L / 16;
  return L % 16 == 0 && (r1 == 3 || r1 == 5 || r1 == 6 || r1 == 10 || r1 == 12 || r1 == 20);
}

cudaError_t launch_dst(const GemmDesc* d_descs, int ndesc, int n, int64_t maxN, bool kcontig, const Bufs& bufs,
                       cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  const int L = 2 * (n + 1);
#define DL(A, B) return kcontig ? dst_launch<A, B, true>(d_descs, ndesc, maxN, bufs, st) \
                                : dst_launch<A, B, false>(d_descs, ndesc, maxN, bufs, st)
  switch (L) {  // contiguous columns: warp-autonomous kernel; strided columns: CTA tiles (coalescing)
    case 16: DL(4, 4);
    case 32:
      if (kcontig) return dstw_launch<4, 8>(d_descs, ndesc, maxN, bufs, st);
      return dst_launch<4, 8, false>(d_descs, ndesc, maxN, bufs, st);
    case 64:
      if (kcontig) return dstw_launch<8, 8>(d_descs, ndesc, maxN, bufs, st);
      return dst_launch<8, 8, false>(d_descs, ndesc, maxN, bufs, st);
    case 128:
      if (kcontig) return dstw_launch<8, 16>(d_descs, ndesc, maxN, bufs, st);
      return dst_launch<8, 16, false>(d_descs, ndesc, maxN, bufs, st);
    case 256:
      if (kcontig) return dstw_launch<16, 16>(d_descs, ndesc, maxN, bufs, st);
      return dst_launch<16, 16, false>(d_descs, ndesc, maxN, bufs, st);
    case 512: DL(16, 32);
#define DM(R1)                                                                        \
  case 16 * R1:                                                                       \
    if (kcontig) return dstw_launch<R1, 16>(d_descs, ndesc, maxN, bufs, st);          \
    return dst_launch<R1, 16, false>(d_descs, ndesc, maxN, bufs, st);
    DM(3) DM(5) DM(6) DM(10) DM(12) DM(20)
#undef DM
    default: return cudaErrorInvalidValue;
  }
#undef DL
}

// Tensor map of descriptor D's input (strided columns of the y sine passes): 2 N2 doubles x K
// rows x N1 planes, box = one CPB-column tile of all rows of one plane.  false when the layout
// is not that one (columns contiguous within a plane, output rows strided) or encoding fails.
bool dst_tma_encode(const GemmDesc& D, int n, const Bufs& bufs, void* map_out) {
  EncodeTiledFn enc = encode_tiled();
  const int L = 2 * (n + 1);
  const int R2 = L == 16 ? 4 : L == 32 || L == 64 ? 8 : L == 512 ? 32 : 16;
  const int CPB = DST_THREADS / R2;
  if (!enc || D.sB2 != 1 || D.sCi == 1 || D.K != n || D.N1 < 1) return false;
  if ((D.sBj * 16) % 16 || (D.sB1 * 16) % 16) return false;
  void* base = reinterpret_cast<char*>(bufs.p[D.b_buf]) + D.b_off * 16;
  if (reinterpret_cast<uintptr_t>(base) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)2 * D.N2, (cuuint64_t)n, (cuuint64_t)D.N1};
  cuuint64_t strides[2] = {(cuuint64_t)D.sBj * 16, (cuuint64_t)D.sB1 * 16};
  cuuint32_t box[3] = {(cuuint32_t)(2 * CPB), (cuuint32_t)n, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (D.N1 > 1 && D.sB1 < D.sBj * (int64_t)n) return false;  // planes must not overlap the rows
  return enc(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool dst_tma_supported(int n) {
  // measured (profiles/r02/experiments/dstt_*): L = 256 (C4's 127-node blocks) 3.35 -> 3.14 ms
  // per step; L = 320 (C4j) and L = 32 (C3) slightly slower than the cp.async tiles of k_dst
  const int L = 2 * (n + 1);
  return encode_tiled() != nullptr && L == 256;
}

cudaError_t launch_dst_tma(const GemmDesc* d_descs, const void* d_maps, int ndesc, int n, int maxN2, int maxN1,
                           const Bufs& bufs, cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  switch (2 * (n + 1)) {
    case 32: return dstt_launch<4, 8>(d_descs, d_maps, ndesc, maxN2, maxN1, bufs, st);
    case 64: return dstt_launch<8, 8>(d_descs, d_maps, ndesc, maxN2, maxN1, bufs, st);
    case 128: return dstt_launch<8, 16>(d_descs, d_maps, ndesc, maxN2, maxN1, bufs, st);
    case 256: return dstt_launch<16, 16>(d_descs, d_maps, ndesc, maxN2, maxN1, bufs, st);
#define DT(R1) case 16 * R1: return dstt_launch<R1, 16>(d_descs, d_maps, ndesc, maxN2, maxN1, bufs, st);
    DT(3) DT(5) DT(6) DT(10) DT(12) DT(20)
#undef DT
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfds
