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
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "lfds_internal.h"

namespace lfds {
namespace {

struct zc2 {
  double x, y;
};
__device__ __forceinline__ zc2 zadd(zc2 a, zc2 b) { return zc2{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ zc2 zsub(zc2 a, zc2 b) { return zc2{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ zc2 zmul(zc2 a, zc2 b) {
  return zc2{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}

// in-register radix-2 DIT FFT (forward, e^{-2 pi i k n / R}); all indices compile-time;
// twiddles W_len^j = W_L^{j L/len} are warp-uniform broadcast reads of the W_L table
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
#pragma unroll
  for (int len = 2; len <= R; len <<= 1) {
#pragma unroll
    for (int i = 0; i < R; i += len) {
#pragma unroll
      for (int j = 0; j < len / 2; ++j) {
        const double2 w2 = twl[j * (L / len)];
        const zc2 w{w2.x, w2.y};
        const zc2 u = v[i + j], t = zmul(w, v[i + j + len / 2]);
        v[i + j] = zadd(u, t);
        v[i + j + len / 2] = zsub(u, t);
      }
    }
  }
}

constexpr int DST_THREADS = 128;  // 8 columns per CTA at L = 256: small CTAs, many resident per SM

__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0));
}

template <int R1, int R2, bool KCONTIG>
__global__ void __launch_bounds__(DST_THREADS) k_dst(const GemmDesc* __restrict__ descs, Bufs bufs) {
  constexpr int L = R1 * R2, N = L / 2;
  constexpr int CPB = DST_THREADS / R2;      // columns per CTA
  constexpr int LDT = CPB + 1;               // tile row stride (complex)
  constexpr int LDE = R2 + 1;                // exchange row stride
  extern __shared__ __align__(16) double2 dsm[];
  // buffer: tile [N-1][LDT] (load, later output staging) aliased with exchange [CPB][R1][LDE]
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
  const int col = tid / R2, t = tid % R2;
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
  fft_reg<R1, L>(a, twl);
#pragma unroll
  for (int k1 = 1; k1 < R1; ++k1) {
    const double2 w = twl[(t * k1) % L];
    a[k1] = zmul(a[k1], zc2{w.x, w.y});
  }
  __syncthreads();  // tile fully consumed
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) ex[(col * R1 + k1) * LDE + t] = make_double2(a[k1].x, a[k1].y);
  __syncthreads();
  // ---- step 3: thread k1 = t < R1: R2-point FFT over n2 -> Y[k1 + R1 k2], keep k < N
  zc2 b[R2];
  if (t < R1) {
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      const double2 w = ex[(col * R1 + t) * LDE + n2];
      b[n2] = zc2{w.x, w.y};
    }
    fft_reg<R2, L>(b, twl);
  }
  __syncthreads();  // exchange consumed; reuse as output tile[c][col]
  const double half = 0.5 * D.scale;
  if (t < R1) {
#pragma unroll
    for (int k2 = 0; k2 < R2 / 2; ++k2) {
      const int k = t + R1 * k2;
      if (k >= 1 && k < N) tile[(k - 1) * LDT + col] = make_double2(-half * b[k2].y, half * b[k2].x);  // (i/2) Y
    }
  }
  __syncthreads();
  if (D.sCi == 1) {  // output column contiguous
    for (int idx = tid; idx < n * CPB; idx += DST_THREADS) {
      const int cc = idx / n, c = idx - cc * n;
      const int64_t o = colC[cc];
      if (o >= 0) C[o + c] = tile[c * LDT + cc];
    }
  } else {
    for (int idx = tid; idx < n * CPB; idx += DST_THREADS) {
      const int c = idx / CPB, cc = idx - c * CPB;
      const int64_t o = colC[cc];
      if (o >= 0) C[o + (int64_t)c * D.sCi] = tile[c * LDT + cc];
    }
  }
}

template <int R1, int R2, bool KC>
cudaError_t dst_launch(const GemmDesc* d, int ndesc, int64_t maxN, const Bufs& bufs, cudaStream_t st) {
  constexpr int L = R1 * R2, N = L / 2, CPB = DST_THREADS / R2;
  const size_t tile = (size_t)(N - 1) * (CPB + 1) * sizeof(double2);
  const size_t ex = (size_t)CPB * R1 * (R2 + 1) * sizeof(double2);
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

}  // namespace

bool dst_supported(int n) {
  const int L = 2 * (n + 1);
  return L == 16 || L == 32 || L == 64 || L == 128 || L == 256 || L == 512;
}

cudaError_t launch_dst(const GemmDesc* d_descs, int ndesc, int n, int64_t maxN, bool kcontig, const Bufs& bufs,
                       cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  const int L = 2 * (n + 1);
#define DL(A, B) return kcontig ? dst_launch<A, B, true>(d_descs, ndesc, maxN, bufs, st) \
                                : dst_launch<A, B, false>(d_descs, ndesc, maxN, bufs, st)
  switch (L) {
    case 16: DL(4, 4);
    case 32: DL(4, 8);
    case 64: DL(8, 8);
    case 128: DL(8, 16);
    case 256: DL(16, 16);
    case 512: DL(16, 32);
    default: return cudaErrorInvalidValue;
  }
#undef DL
}

}  // namespace lfds
