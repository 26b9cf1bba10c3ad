// Vector kernels of the preconditioned Krylov solve for horizontally heterogeneous media
// (lfds_gmres: the layered-medium fast solver as the preconditioner of an
// iterative method for media with embedded inhomogeneities).
//
// With lambda_ijk = lambda + dlam_ijk the heterogeneous operator is A_het = A + diag(dlam) M
// (the lambda term of Eq. (fd) carries the control volume M = hx^ hy^ hz^), so with the fast
// solver S = A^{-1} M (f-units in, u out) the right-preconditioned operator is exactly
//     M^{-1} A_het S = I + diag(dlam) S          (Lippmann-Schwinger / FDIE form)
// and one Arnoldi step needs one fast solve and the pointwise k_fdie — no stencil matvec.
// k_dots / k_maxpy are the (classical Gram-Schmidt) inner products and updates over up to 65
// basis vectors; k_dots writes per-CTA partial sums that the host adds in CTA order, so the
// iteration is deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "lfds_internal.h"

namespace lfds {
namespace {

constexpr int KT = 256;  // threads per CTA

// w = v + dlam .* s  (v == NULL: w = dlam .* s; out may alias v)
__global__ void k_fdie(int64_t n, const double2* __restrict__ v, const double2* __restrict__ dlam,
                       const double2* __restrict__ s, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    const double2 a = v ? v[i] : make_double2(0, 0), d = dlam[i], b = s[i];
    out[i] = make_double2(a.x + fma(d.x, b.x, -d.y * b.y), a.y + fma(d.x, b.y, d.y * b.x));
  }
}

// r = f - (y + dlam .* s)
__global__ void k_fdie_res(int64_t n, const double2* __restrict__ f, const double2* __restrict__ y,
                           const double2* __restrict__ dlam, const double2* __restrict__ s, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    const double2 a = y[i], d = dlam[i], b = s[i], g = f[i];
    out[i] = make_double2(g.x - a.x - fma(d.x, b.x, -d.y * b.y), g.y - a.y - fma(d.x, b.y, d.y * b.x));
  }
}

// partial[blk][i] = sum over this CTA's elements of conj(V_i) w, i < cnt (8 vectors per sweep);
// with_self: also conj(w) w in slot cnt (the norm before orthogonalisation, same sweep)
__global__ void k_dots(int64_t n, int cnt, const double2* __restrict__ V, int64_t vstride,
                       const double2* __restrict__ w, double2* partial, int with_self) {
  constexpr int QV = 8;  // vectors per sweep over w
  __shared__ double2 red[KT / 32][QV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tot = cnt + (with_self ? 1 : 0);
  for (int i0 = 0; i0 < tot; i0 += QV) {
    double2 acc[QV];
#pragma unroll
    for (int q = 0; q < QV; ++q) acc[q] = make_double2(0, 0);
    for (int64_t e = (int64_t)blockIdx.x * KT + threadIdx.x; e < n; e += (int64_t)gridDim.x * KT) {
      const double2 b = w[e];
#pragma unroll
      for (int q = 0; q < QV; ++q) {
        if (i0 + q < tot) {
          const double2 a = i0 + q < cnt ? V[(int64_t)(i0 + q) * vstride + e] : b;
          acc[q].x = fma(a.x, b.x, fma(a.y, b.y, acc[q].x));   // conj(a) b
          acc[q].y = fma(a.x, b.y, fma(-a.y, b.x, acc[q].y));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < QV; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
        acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
      }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < QV; ++q) red[warp][q] = acc[q];
    __syncthreads();
    if (threadIdx.x < QV && i0 + (int)threadIdx.x < tot) {
      double2 s = red[0][threadIdx.x];
      for (int wi = 1; wi < KT / 32; ++wi) {
        s.x += red[wi][threadIdx.x].x;
        s.y += red[wi][threadIdx.x].y;
      }
      partial[(int64_t)blockIdx.x * 80 + i0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// w += sum_i coef_i V_i   (coef on the device, cnt <= 80)
__global__ void k_maxpy(int64_t n, int cnt, const double2* __restrict__ V, int64_t vstride,
                        const double2* __restrict__ coef, double2* w) {
  __shared__ double2 c[80];
  for (int i = threadIdx.x; i < cnt; i += KT) c[i] = coef[i];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * KT + threadIdx.x; e < n; e += (int64_t)gridDim.x * KT) {
    double2 acc = w[e];
    for (int i = 0; i < cnt; ++i) {
      const double2 a = V[(int64_t)i * vstride + e], k = c[i];
      acc.x = fma(k.x, a.x, fma(-k.y, a.y, acc.x));
      acc.y = fma(k.x, a.y, fma(k.y, a.x, acc.y));
    }
    w[e] = acc;
  }
}

// w += sum_i coef_i V_i, and partial[blk][0] = this CTA's part of ||w||^2 after the update
__global__ void k_maxpy_norm(int64_t n, int cnt, const double2* __restrict__ V, int64_t vstride,
                             const double2* __restrict__ coef, double2* w, double2* partial) {
  __shared__ double2 c[80];
  __shared__ double red[KT / 32];
  for (int i = threadIdx.x; i < cnt; i += KT) c[i] = coef[i];
  __syncthreads();
  double nrm = 0;
  for (int64_t e = (int64_t)blockIdx.x * KT + threadIdx.x; e < n; e += (int64_t)gridDim.x * KT) {
    double2 acc = w[e];
    for (int i = 0; i < cnt; ++i) {
      const double2 a = V[(int64_t)i * vstride + e], k = c[i];
      acc.x = fma(k.x, a.x, fma(-k.y, a.y, acc.x));
      acc.y = fma(k.x, a.y, fma(k.y, a.x, acc.y));
    }
    w[e] = acc;
    nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sacc = 0;
    for (int wi = 0; wi < KT / 32; ++wi) sacc += red[wi];
    partial[(int64_t)blockIdx.x * 80] = make_double2(sacc, 0);
  }
}

// out = alpha w
__global__ void k_scale(int64_t n, double2 alpha, const double2* __restrict__ w, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    const double2 a = w[i];
    out[i] = make_double2(fma(alpha.x, a.x, -alpha.y * a.y), fma(alpha.x, a.y, alpha.y * a.x));
  }
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n + KT - 1) / KT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 8));
}

}  // namespace

cudaError_t launch_fdie(int64_t n, const double2* v, const double2* dlam, const double2* s, double2* out,
                        cudaStream_t st) {
  k_fdie<<<grid_for(n), KT, 0, st>>>(n, v, dlam, s, out);
  return cudaGetLastError();
}
cudaError_t launch_fdie_res(int64_t n, const double2* f, const double2* y, const double2* dlam, const double2* s,
                            double2* out, cudaStream_t st) {
  k_fdie_res<<<grid_for(n), KT, 0, st>>>(n, f, y, dlam, s, out);
  return cudaGetLastError();
}
cudaError_t launch_dots(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* w, double2* partial,
                        cudaStream_t st, int with_self) {
  if (cnt < 1 || cnt + (with_self ? 1 : 0) > 80) return cudaErrorInvalidValue;
  k_dots<<<KRYLOV_DOT_BLOCKS, KT, 0, st>>>(n, cnt, V, vstride, w, partial, with_self);
  return cudaGetLastError();
}
cudaError_t launch_maxpy(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* coef, double2* w,
                         cudaStream_t st) {
  if (cnt < 1 || cnt > 80) return cudaErrorInvalidValue;
  k_maxpy<<<grid_for(n), KT, 0, st>>>(n, cnt, V, vstride, coef, w);
  return cudaGetLastError();
}
cudaError_t launch_maxpy_norm(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* coef, double2* w,
                              double2* partial, cudaStream_t st) {
  if (cnt < 1 || cnt > 80) return cudaErrorInvalidValue;
  k_maxpy_norm<<<KRYLOV_DOT_BLOCKS, KT, 0, st>>>(n, cnt, V, vstride, coef, w, partial);
  return cudaGetLastError();
}
cudaError_t launch_scale(int64_t n, double2 alpha, const double2* w, double2* out, cudaStream_t st) {
  k_scale<<<grid_for(n), KT, 0, st>>>(n, alpha, w, out);
  return cudaGetLastError();
}

}  // namespace lfds
