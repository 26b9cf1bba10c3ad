// sm_100a kernels of the blocked separable Helmholtz solve (arXiv 1909.01299).
//
//  k_gemm          strided batched complex contraction on FP64 ALUs: every transform of the
//                  f64 (real, LFDS_F64) plans; complex plans run their transforms on the tensor
//                  pipe (lfds_xform.cu) and the sine kernels (lfds_dst.cu).
//  (z-solves of steps 2, 5 and 6: lfds_zsolve.cu)
//  k_iface_res     step 4: residual b - A v on the interface planes.
//  k_write_iface   u = w on the interface planes (last sentence).
//  k_residual      r = M f - A u (Eq. (fd)), fp64 or double-double (refinement, reading R13).
#include "lfds_internal.h"

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace lfds {

// ---------------------------------------------------------------- complex helpers
struct cplx {
  double x, y;
};
__device__ __forceinline__ cplx mk(double a, double b) { return cplx{a, b}; }
__device__ __forceinline__ cplx ld(const double2* p) {
  double2 v = __ldg(p);
  return cplx{v.x, v.y};
}
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return cplx{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return cplx{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cplx operator-(cplx a) { return cplx{-a.x, -a.y}; }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
  return cplx{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ cplx operator*(double s, cplx b) { return cplx{s * b.x, s * b.y}; }
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {  // a*b + c
  return cplx{fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
__device__ __forceinline__ cplx cinv(cplx a) {
  double n = 1.0 / fma(a.x, a.x, a.y * a.y);
  return cplx{a.x * n, -a.y * n};
}
__device__ __forceinline__ double cabs1(cplx a) { return fabs(a.x) + fabs(a.y); }
// reciprocal from the MUFU.RCP64H seed (~20 bits) and two Newton steps (full fp64 accuracy,
// <= 1 ulp): 5 instructions instead of the IEEE division sequence with its slow-path branch
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ cplx cinv_fast(cplx a) {
  const double n = fast_rcp(fma(a.x, a.x, a.y * a.y));
  return cplx{a.x * n, -a.y * n};
}
__device__ __forceinline__ cplx shfl_up(cplx v, int d) {
  return cplx{__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d)};
}
__device__ __forceinline__ cplx shfl_down(cplx v, int d) {
  return cplx{__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d)};
}

// minimum of positive doubles through their ordered bit patterns
__device__ __forceinline__ void atomic_min_pos(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------- generic contraction
// C(i, n) (+)= sum_j A(i, j) B(j, n); 256 threads, tile TM x TN outputs, TK-deep chunks.
constexpr int GTM = 32, GTN = 64, GTK = 16;

__global__ void __launch_bounds__(256) k_gemm(const GemmDesc* __restrict__ descs, Bufs bufs) {
  const GemmDesc& D = descs[blockIdx.z];
  const int M = D.M, K = D.K, N2 = D.N2;
  const int64_t N = (int64_t)D.N1 * N2;
  const int i0 = blockIdx.y * GTM;
  const int64_t n0 = (int64_t)blockIdx.x * GTN;
  if (i0 >= M || n0 >= N) return;
  __shared__ double2 smem[(GTK * (GTM + 1) + GTK * (GTN + 1)) > (GTM * (GTN + 1)) ? (GTK * (GTM + 1) + GTK * (GTN + 1)) : (GTM * (GTN + 1))];
  double2* As = smem;                       // [GTK][GTM+1]
  double2* Bs = smem + GTK * (GTM + 1);     // [GTK][GTN+1]
  const double2* A = reinterpret_cast<const double2*>(bufs.p[B_TAB]) + D.a_off;
  const bool breal = D.flags & G_BREAL;
  const char* Bb = reinterpret_cast<const char*>(bufs.p[D.b_buf]);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const bool jfast = (D.sBj == 1);
  cplx acc[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = mk(0, 0);

  for (int j0 = 0; j0 < K; j0 += GTK) {
    for (int e = tid; e < GTM * GTK; e += 256) {
      int jj = e % GTK, ii = e / GTK;
      int i = i0 + ii, j = j0 + jj;
      double2 v = make_double2(0, 0);
      if (i < M && j < K) v = __ldg(A + i * D.sAi + j * D.sAj);
      As[jj * (GTM + 1) + ii] = v;
    }
    for (int e = tid; e < GTK * GTN; e += 256) {
      int jj, nn;
      if (jfast) { jj = e % GTK; nn = e / GTK; } else { nn = e % GTN; jj = e / GTN; }
      int64_t n = n0 + nn;
      int j = j0 + jj;
      double2 v = make_double2(0, 0);
      if (n < N && j < K) {
        int64_t n1 = n / N2, n2 = n - n1 * N2;
        int64_t off = D.b_off + (int64_t)j * D.sBj + n1 * D.sB1 + n2 * D.sB2;
        if (breal) v.x = __ldg(reinterpret_cast<const double*>(Bb) + off);
        else v = __ldg(reinterpret_cast<const double2*>(Bb) + off);
      }
      Bs[jj * (GTN + 1) + nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < GTK; ++jj) {
      cplx a0, a1, b[4];
      double2 t = As[jj * (GTM + 1) + ty]; a0 = mk(t.x, t.y);
      t = As[jj * (GTM + 1) + ty + 16]; a1 = mk(t.x, t.y);
#pragma unroll
      for (int q = 0; q < 4; ++q) { t = Bs[jj * (GTN + 1) + tx + 16 * q]; b[q] = mk(t.x, t.y); }
#pragma unroll
      for (int q = 0; q < 4; ++q) { acc[0][q] = cfma(a0, b[q], acc[0][q]); acc[1][q] = cfma(a1, b[q], acc[1][q]); }
    }
    __syncthreads();
  }
  // stage the tile in shared memory, then store with the C-contiguous index fastest
  double2* Cs = smem;  // [GTM][GTN+1]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) Cs[(ty + 16 * a) * (GTN + 1) + tx + 16 * q] = make_double2(acc[a][q].x, acc[a][q].y);
  __syncthreads();
  const bool ifast = (D.sCi == 1);
  const bool creal = D.flags & G_CREAL, accum = D.flags & G_ACCUM;
  char* Cb = reinterpret_cast<char*>(bufs.p[D.c_buf]);
  for (int e = tid; e < GTM * GTN; e += 256) {
    int ii, nn;
    if (ifast) { ii = e % GTM; nn = e / GTM; } else { nn = e % GTN; ii = e / GTN; }
    int i = i0 + ii;
    int64_t n = n0 + nn;
    if (i >= M || n >= N) continue;
    int64_t n1 = n / N2, n2 = n - n1 * N2;
    int64_t off = D.c_off + (int64_t)i * D.sCi + n1 * D.sC1 + n2 * D.sC2;
    double2 v = Cs[ii * (GTN + 1) + nn];
    if (creal) {
      double* c = reinterpret_cast<double*>(Cb) + off;
      *c = accum ? *c + v.x : v.x;
    } else {
      double2* c = reinterpret_cast<double2*>(Cb) + off;
      if (accum) { double2 o = *c; v.x += o.x; v.y += o.y; }
      *c = v;
    }
  }
}

cudaError_t launch_gemm(const GemmDesc* d_descs, int ndesc, int maxM, int maxN, int, const Bufs& bufs,
                        cudaStream_t st) {
  if (ndesc <= 0) return cudaSuccess;
  for (int z0 = 0; z0 < ndesc; z0 += 65535) {
    int nz = ndesc - z0 < 65535 ? ndesc - z0 : 65535;
    dim3 grid((unsigned)((maxN + GTN - 1) / GTN), (unsigned)((maxM + GTM - 1) / GTM), (unsigned)nz);
    k_gemm<<<grid, 256, 0, st>>>(d_descs + z0, bufs);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- step 4 interface residual
// x-plane a (node P): r = b - (1/hx_{P-1}) hy^_q s_k hz^_k v(P-1,q,k) - (1/hx_P) hy^_q s_k hz^_k v(P+1,q,k)
// for q not on a y-interface, r = b on the intersection lines (v = 0 on every neighbour).
// v at the interface-adjacent rows comes from step 3: VX[blk][r][e][k][qpad], VY[blk][r][e][k][ppad].
__device__ __forceinline__ cplx load_f(const void* f, int dtype, int64_t off) {
  if (dtype == 1) return mk(__ldg(reinterpret_cast<const double*>(f) + off), 0.0);
  return ld(reinterpret_cast<const double2*>(f) + off);
}

__global__ void k_iface_res(IfaceRes P, Bufs bufs) {
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  const int* ifx = reinterpret_cast<const int*>(TAB + P.ifx);
  const int* ify = reinterpret_cast<const int*>(TAB + P.ify);
  const int* bx = reinterpret_cast<const int*>(TAB + P.blk_of_x);
  const int* by = reinterpret_cast<const int*>(TAB + P.blk_of_y);
  const int* xlo = reinterpret_cast<const int*>(TAB + P.xlo);
  const int* ylo = reinterpret_cast<const int*>(TAB + P.ylo);
  const void* f = bufs.p[B_F];
  const int nx = P.nx, ny = P.ny, nz = P.nz, R = P.R;
  const int64_t nxplane = (int64_t)P.nifx * R * nz * ny;
  const int64_t total = nxplane + (int64_t)P.nify * R * nz * nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nxplane) {
      const int q = (int)(t % ny);              // 0-based global y index
      int64_t rest = t / ny;
      const int k = (int)(rest % nz); rest /= nz;
      const int r = (int)(rest % R);
      const int a = (int)(rest / R);
      const int Pn = ifx[a];                    // 1-based node
      const int64_t fo = (((int64_t)r * nz + k) * ny + q) * nx + (Pn - 1);
      cplx hh = ld(TAB + P.hhx + Pn - 1) * ld(TAB + P.hhy + q) * ld(TAB + P.hhz + k);
      cplx res = P.with_b ? hh * load_f(f, P.dtype, fo) : mk(0, 0);
      const int jb = by[q];
      if (jb >= 0) {
        const int ql = q + 1 - ylo[jb];
        const cplx wgt = ld(TAB + P.hhy + q) * ld(TAB + P.sig + k) * ld(TAB + P.hhz + k);
        // left block column a, its last row (e=1); right block column a+1, its first row (e=0);
        // with block sharding only the blocks this rank computed contribute
        const int bl = jb * P.nbx + a, br = jb * P.nbx + a + 1;
        if (P.own[bl]) {
          const cplx vl = ld(IF + P.vxo + ((((int64_t)bl * 2 + 1) * R + r) * nz + k) * P.qpad + ql);
          res = res - (cinv(ld(TAB + P.hx + Pn - 1)) * wgt) * vl;
        }
        if (P.own[br]) {
          const cplx vr = ld(IF + P.vxo + ((((int64_t)br * 2 + 0) * R + r) * nz + k) * P.qpad + ql);
          res = res - (cinv(ld(TAB + P.hx + Pn)) * wgt) * vr;
        }
      }
      IF[P.rx + t] = make_double2(res.x, res.y);  // RX[a][r][k][q]
    } else {
      const int64_t u = t - nxplane;
      const int p = (int)(u % nx);
      int64_t rest = u / nx;
      const int k = (int)(rest % nz); rest /= nz;
      const int r = (int)(rest % R);
      const int b = (int)(rest / R);
      const int Qn = ify[b];
      const int ib = bx[p];
      cplx res = mk(0, 0);
      if (ib >= 0) {  // nodes on x-interfaces are owned by RX
        const int64_t fo = (((int64_t)r * nz + k) * ny + (Qn - 1)) * nx + p;
        cplx hh = ld(TAB + P.hhx + p) * ld(TAB + P.hhy + Qn - 1) * ld(TAB + P.hhz + k);
        if (P.with_b) res = hh * load_f(f, P.dtype, fo);
        const int pl = p + 1 - xlo[ib];
        const cplx wgt = ld(TAB + P.hhx + p) * ld(TAB + P.sig + k) * ld(TAB + P.hhz + k);
        const int bb = b * P.nbx + ib, bt = (b + 1) * P.nbx + ib;
        if (P.own[bb]) {
          const cplx vb = ld(IF + P.vyo + ((((int64_t)bb * 2 + 1) * R + r) * nz + k) * P.ppad + pl);
          res = res - (cinv(ld(TAB + P.hy + Qn - 1)) * wgt) * vb;
        }
        if (P.own[bt]) {
          const cplx vt = ld(IF + P.vyo + ((((int64_t)bt * 2 + 0) * R + r) * nz + k) * P.ppad + pl);
          res = res - (cinv(ld(TAB + P.hy + Qn)) * wgt) * vt;
        }
      }
      IF[P.ry + u] = make_double2(res.x, res.y);  // RY[b][r][k][p]
    }
  }
}

cudaError_t launch_iface_residual(const IfaceRes& p, const Bufs& bufs, cudaStream_t st) {
  int64_t total = (int64_t)p.nifx * p.R * p.nz * p.ny + (int64_t)p.nify * p.R * p.nz * p.nx;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  k_iface_res<<<(unsigned)(blocks > 65535 * 16 ? 65535 * 16 : blocks), 256, 0, st>>>(p, bufs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- u = w on the interface planes
__global__ void k_write_iface(int nx, int ny, int nz, int R, int dtype, int nifx, int nify, int64_t ifxo,
                              int64_t ifyo, int64_t wx, int64_t wy, Bufs bufs, const int* __restrict__ wmask,
                              int64_t bxo, int64_t byo, int nbx, int nby, int rank0) {
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* IF = reinterpret_cast<const double2*>(bufs.p[B_IF]);
  const int* ifx = reinterpret_cast<const int*>(TAB + ifxo);
  const int* ify = reinterpret_cast<const int*>(TAB + ifyo);
  const int* bx_of = reinterpret_cast<const int*>(TAB + bxo);  // block column of node p (-1: interface)
  const int* by_of = reinterpret_cast<const int*>(TAB + byo);
  void* u = bufs.p[B_U];
  const int64_t nxp = (int64_t)nifx * R * nz * ny;
  const int64_t total = nxp + (int64_t)nify * R * nz * nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t uo;
    double2 v;
    if (t < nxp) {
      const int q = (int)(t % ny);
      int64_t rest = t / ny;
      const int k = (int)(rest % nz); rest /= nz;
      const int r = (int)(rest % R);
      const int a = (int)(rest / R);
      if (wmask) {
        const int j = by_of[q];
        if (j < 0 ? !rank0 : !wmask[a * nby + j]) continue;
      }
      uo = (((int64_t)r * nz + k) * ny + q) * nx + (ifx[a] - 1);
      v = IF[wx + t];
    } else {
      const int64_t s = t - nxp;
      const int p = (int)(s % nx);
      int64_t rest = s / nx;
      const int k = (int)(rest % nz); rest /= nz;
      const int r = (int)(rest % R);
      const int b = (int)(rest / R);
      // intersection lines are written by the x-plane values only
      bool on_x = false;
      for (int a = 0; a < nifx; ++a) on_x |= (ifx[a] - 1 == p);
      if (on_x) continue;
      if (wmask && !wmask[nifx * nby + b * nbx + bx_of[p]]) continue;
      uo = (((int64_t)r * nz + k) * ny + (ify[b] - 1)) * nx + p;
      v = IF[wy + s];
    }
    if (dtype == 1) reinterpret_cast<double*>(u)[uo] = v.x;
    else reinterpret_cast<double2*>(u)[uo] = v;
  }
}

cudaError_t launch_write_iface_u(int nx, int ny, int nz, int R, int dtype, int nifx, int nify, int64_t ifx,
                                 int64_t ify, int64_t wx, int64_t wy, const Bufs& bufs, cudaStream_t st,
                                 const int* wmask, int64_t bxo, int64_t byo, int nbx, int nby, int rank0) {
  int64_t total = (int64_t)nifx * R * nz * ny + (int64_t)nify * R * nz * nx;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  k_write_iface<<<(unsigned)(blocks > 1048576 ? 1048576 : blocks), 256, 0, st>>>(
      nx, ny, nz, R, dtype, nifx, nify, ifx, ify, wx, wy, bufs, wmask, bxo, byo, nbx, nby, rank0);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- residual (fp64 / double-double)
// double-double primitives (error-free transformations with FMA)
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return dd{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  double lo = s.lo + a.lo + b.lo;
  double hi = s.hi + lo;
  return dd{hi, lo - (hi - s.hi)};
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, fma(a.lo, b.hi, e));
  double hi = p + e;
  return dd{hi, e - (hi - p)};
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
struct zdd {
  dd x, y;
};
__device__ __forceinline__ zdd zadd(zdd a, zdd b) { return zdd{dd_add(a.x, b.x), dd_add(a.y, b.y)}; }
__device__ __forceinline__ zdd zsub(zdd a, zdd b) { return zdd{dd_add(a.x, dd_neg(b.x)), dd_add(a.y, dd_neg(b.y))}; }
__device__ __forceinline__ zdd zmul(zdd a, zdd b) {
  return zdd{dd_add(dd_mul(a.x, b.x), dd_neg(dd_mul(a.y, b.y))), dd_add(dd_mul(a.x, b.y), dd_mul(a.y, b.x))};
}
__device__ __forceinline__ zdd zfrom(cplx a) { return zdd{dd{a.x, 0}, dd{a.y, 0}}; }
struct ResParams {
  int nx, ny, nz, R, dtype, dd, has_f, to_f;
  int64_t hx, hy, hz, hhx, hhy, hhz, sig, sige;
  double2 lam;
  int64_t rxd, ryd, szd;  // double-double node tables [n][cl, cr] (see k_residual), 2 slots per value
};

__device__ __forceinline__ cplx load_u(const void* u, int dtype, int64_t off) {
  if (dtype == 1) return mk(reinterpret_cast<const double*>(u)[off], 0.0);
  double2 v = reinterpret_cast<const double2*>(u)[off];
  return mk(v.x, v.y);
}

__device__ __forceinline__ zdd zmul_zd(zdd a, cplx b) {  // dd x double complex
  auto m = [](dd x, double y) {
    const double p = x.hi * y;
    const double e = fma(x.hi, y, -p) + x.lo * y;
    const double hi = p + e;
    return dd{hi, e - (hi - p)};
  };
  return zdd{dd_add(m(a.x, b.x), dd_neg(m(a.y, b.y))), dd_add(m(a.x, b.y), m(a.y, b.x))};
}

// One thread per (i, j) column of a z-chunk: grid (x-tiles of 128, y, r * nchunks + chunk); the
// thread marches k through its chunk of RZ_CHUNK planes with u(k-1), u(k), u(k+1) in registers,
// so u is read from HBM about once (the x / y neighbours of a plane come from L1 / L2) and the
// norms are reduced per column.  The double-double path evaluates the residual in f-units,
// r_f = f - (A u)/V with V = hx^ hy^ hz^:
//   (A u)/V = sigma_k [cxr (u_{i+1} - u_i) - cxl (u_i - u_{i-1}) + cyr (..) - cyl (..)]
//           + czr (u_{k+1} - u_k) - czl (u_k - u_{k-1}) + lambda u_i,
// cxl_i = 1/(h_{i-1} hx^_i), cxr_i = 1/(h_i hx^_i), czl_k = sigma_{k-1/2}/(h_{k-1} hz^_k), ...
// from the plan's long-double tables (Eq. (fd) divided by the control volume, term by term).
constexpr int RZ_CHUNK = 32;
__global__ void __launch_bounds__(128) k_residual(ResParams P, const void* __restrict__ u, const void* __restrict__ f,
                                                  double2* __restrict__ rout, double* norms, Bufs bufs) {
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const int nx = P.nx, ny = P.ny, nz = P.nz;
  const int nch = (nz + RZ_CHUNK - 1) / RZ_CHUNK;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  const int r = blockIdx.z / nch, kc = blockIdx.z - r * nch;
  const int kb = kc * RZ_CHUNK, ke = min(nz, kb + RZ_CHUNK);
  const int64_t plane = (int64_t)nx * ny;
  double acc_r = 0, acc_b = 0;
  // every lane runs the loop (the x neighbours of a plane come from the neighbouring lanes'
  // registers by shuffles); lanes past the row end only take part in the shuffles
  const bool ok = i < nx;
  const int lane = threadIdx.x & 31;
  {
    const int ii = ok ? i : nx - 1;
    const int64_t col = (int64_t)r * nz * plane + (int64_t)j * nx + ii;
    const cplx cx = ld(TAB + P.hhx + ii), cy = ld(TAB + P.hhy + j);
    const cplx lam = mk(P.lam.x, P.lam.y);
    cplx ub = kb > 0 ? load_u(u, P.dtype, col + (int64_t)(kb - 1) * plane) : mk(0, 0);
    cplx uc = load_u(u, P.dtype, col + (int64_t)kb * plane);
    for (int k = kb; k < ke; ++k) {
      const int64_t t = col + (int64_t)k * plane;
      const cplx ut = k < nz - 1 ? load_u(u, P.dtype, t + plane) : mk(0, 0);
      cplx ul = mk(__shfl_up_sync(0xffffffffu, uc.x, 1), __shfl_up_sync(0xffffffffu, uc.y, 1));
      cplx ur = mk(__shfl_down_sync(0xffffffffu, uc.x, 1), __shfl_down_sync(0xffffffffu, uc.y, 1));
      if (lane == 0) ul = i > 0 && ok ? load_u(u, P.dtype, t - 1) : mk(0, 0);
      if (lane == 31 || i >= nx - 1) ur = i < nx - 1 ? load_u(u, P.dtype, t + 1) : mk(0, 0);
      const cplx us = j > 0 ? load_u(u, P.dtype, t - nx) : mk(0, 0);
      const cplx un = j < ny - 1 ? load_u(u, P.dtype, t + nx) : mk(0, 0);
      const cplx cz = ld(TAB + P.hhz + k);
      const cplx sg = ld(TAB + P.sig + k);
      const cplx fv = P.has_f ? load_f(f, P.dtype, t) : mk(0, 0);
      const cplx V = cx * cy * cz;
      cplx res, bnorm;
      if (!P.dd) {
        // fp64: the same f-units evaluation from the per-node stencil tables (their leading
        // doubles), no per-point reciprocals
        auto t64 = [&](int64_t off, int n, int e) {
          const double2 a = __ldg(TAB + off + 4 * n + 2 * e), b = __ldg(TAB + off + 4 * n + 2 * e + 1);
          return mk(a.x, b.x);
        };
        const cplx hx = (ur - uc) * t64(P.rxd, i, 1) - (uc - ul) * t64(P.rxd, i, 0);
        const cplx hy = (un - uc) * t64(P.ryd, j, 1) - (uc - us) * t64(P.ryd, j, 0);
        const cplx hz = (ut - uc) * t64(P.szd, k, 1) - (uc - ub) * t64(P.szd, k, 0);
        const cplx Lu = sg * (hx + hy) + hz + lam * uc;
        const cplx rf = fv - Lu;
        res = P.to_f ? rf : rf * V;
        bnorm = fv * V;
      } else {
        auto tdd = [&](int64_t off, int n, int e) {  // node table: [n][cl, cr], 2 slots each
          const double2 a = __ldg(TAB + off + 4 * n + 2 * e), b = __ldg(TAB + off + 4 * n + 2 * e + 1);
          return zdd{dd{a.x, a.y}, dd{b.x, b.y}};
        };
        const zdd Uc = zfrom(uc);
        zdd h = zsub(zmul(zsub(zfrom(ur), Uc), tdd(P.rxd, i, 1)), zmul(zsub(Uc, zfrom(ul)), tdd(P.rxd, i, 0)));
        h = zadd(h, zsub(zmul(zsub(zfrom(un), Uc), tdd(P.ryd, j, 1)), zmul(zsub(Uc, zfrom(us)), tdd(P.ryd, j, 0))));
        zdd Lu = zmul_zd(h, sg);
        Lu = zadd(Lu, zsub(zmul(zsub(zfrom(ut), Uc), tdd(P.szd, k, 1)), zmul(zsub(Uc, zfrom(ub)), tdd(P.szd, k, 0))));
        Lu = zadd(Lu, zmul_zd(zfrom(uc), lam));
        const zdd rf = zsub(zfrom(fv), Lu);
        const cplx rfc = mk(rf.x.hi + rf.x.lo, rf.y.hi + rf.y.lo);
        res = P.to_f ? rfc : rfc * V;
        bnorm = fv * V;
      }
      if (ok) {
        if (rout) rout[t] = make_double2(res.x, res.y);
        const cplx rb = P.to_f ? res * V : res;
        acc_r += rb.x * rb.x + rb.y * rb.y;
        acc_b += bnorm.x * bnorm.x + bnorm.y * bnorm.y;
      }
      ub = uc;
      uc = ut;
    }
  }
  if (norms) {  // warp sums, one atomic pair per warp and chunk
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc_r += __shfl_xor_sync(0xffffffffu, acc_r, o);
      acc_b += __shfl_xor_sync(0xffffffffu, acc_b, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(norms + 2 * r, acc_r);
      atomicAdd(norms + 2 * r + 1, acc_b);
    }
  }
}

cudaError_t launch_residual(int nx, int ny, int nz, int R, int dtype, int ddm, int has_f, int64_t hx, int64_t hy,
                            int64_t hz, int64_t hhx, int64_t hhy, int64_t hhz, int64_t sig, int64_t sige, double2 lam,
                            const int64_t* ddtabs, const void* u, const void* f, double2* r, int to_f_units,
                            double* d_norms, const Bufs& bufs, cudaStream_t st) {
  ResParams P{nx, ny, nz, R, dtype, ddm, has_f, to_f_units, hx, hy, hz, hhx, hhy, hhz, sig, sige, lam,
              ddtabs[0], ddtabs[1], ddtabs[2]};
  const int64_t nch = (nz + RZ_CHUNK - 1) / RZ_CHUNK;
  if (nch * R > 65535 || ny > 65535) return cudaErrorInvalidValue;
  k_residual<<<dim3((unsigned)((nx + 127) / 128), (unsigned)ny, (unsigned)(nch * R)), 128, 0, st>>>(P, u, f, r, d_norms,
                                                                                                    bufs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- u += delta
__global__ void k_axpy(int64_t n, int dtype, const double2* __restrict__ dlt, void* u) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double2 d = dlt[t];
    if (dtype == 1) reinterpret_cast<double*>(u)[t] += d.x;
    else {
      double2* p = reinterpret_cast<double2*>(u) + t;
      double2 o = *p;
      *p = make_double2(o.x + d.x, o.y + d.y);
    }
  }
}

cudaError_t launch_axpy_u(int64_t n, int dtype, const double2* delta, void* u, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_axpy<<<(unsigned)blocks, 256, 0, st>>>(n, dtype, delta, u);
  return cudaGetLastError();
}

__global__ void k_fill_one(double* p) { *p = 1.0; }
cudaError_t launch_fill_minpiv(double* p, cudaStream_t st) {
  k_fill_one<<<1, 1, 0, st>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- step-5 folds
// A palindromic axis (h_t = h_{N-t}) has only even and odd global modes, W[N-1-q][l] = +-W[q][l]
// exactly, so sum_q W[q][l] x_q = sum_{q < ceil(N/2)} W[q][l] (x_q + x_{N-1-q}) for even l (the
// middle row once) and sum_{q < floor(N/2)} W[q][l] (x_q - x_{N-1-q}) for odd l: half-length
// contractions of the folded data.  k_fold forms the folds, k_unfold recombines the two halves.
__global__ void k_fold(int64_t rows, int N, const double2* __restrict__ x, double2* __restrict__ s) {
  const int nh = N / 2, ks = N - nh;
  double2* a = s + rows * ks;
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const double2* xr = x + i * N;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < ks; q += gridDim.x * blockDim.x) {
      const double2 u = xr[q];
      if (q < nh) {
        const double2 v = xr[N - 1 - q];
        s[i * ks + q] = make_double2(u.x + v.x, u.y + v.y);
        a[i * nh + q] = make_double2(u.x - v.x, u.y - v.y);
      } else {
        s[i * ks + q] = u;  // middle row of an odd N
      }
    }
  }
}
__global__ void k_unfold(int64_t rows, int N, const double2* __restrict__ s, double2* __restrict__ w) {
  const int nh = N / 2, ks = N - nh;
  const double2* o = s + rows * ks;
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    double2* wr = w + i * N;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < ks; q += gridDim.x * blockDim.x) {
      const double2 e = s[i * ks + q];
      if (q < nh) {
        const double2 d = o[i * nh + q];
        wr[q] = make_double2(e.x + d.x, e.y + d.y);
        wr[N - 1 - q] = make_double2(e.x - d.x, e.y - d.y);
      } else {
        wr[q] = e;
      }
    }
  }
}

cudaError_t launch_fold(bool forward, int64_t rows, int N, int64_t plane, int64_t fold, const Bufs& bufs,
                        cudaStream_t st) {
  if (rows <= 0 || N < 1) return cudaSuccess;
  double2* IF = reinterpret_cast<double2*>(bufs.p[B_IF]);
  const int ks = N - N / 2;
  const dim3 grid((unsigned)((ks + 127) / 128), (unsigned)std::min<int64_t>(rows, 65535));
  if (forward) k_fold<<<grid, 128, 0, st>>>(rows, N, IF + plane, IF + fold);
  else k_unfold<<<grid, 128, 0, st>>>(rows, N, IF + fold, IF + plane);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- multi-level glue (lfds_ml.cpp)
__global__ void k_ml_gather(const double2* __restrict__ r, int nx, int ny, int nz, const int* __restrict__ ifx,
                            int nifx, const int* __restrict__ ify, int nify, double2* __restrict__ rx,
                            double2* __restrict__ ry) {
  const int64_t nX = (int64_t)nifx * nz * ny, total = nX + (int64_t)nify * nz * nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nX) {
      const int q = (int)(t % ny);
      const int64_t rest = t / ny;
      const int k = (int)(rest % nz), a = (int)(rest / nz);
      rx[t] = r[((int64_t)k * ny + q) * nx + ifx[a] - 1];
    } else {
      const int64_t u = t - nX;
      const int p = (int)(u % nx);
      const int64_t rest = u / nx;
      const int k = (int)(rest % nz), b = (int)(rest / nz);
      bool on_x = false;
      for (int a = 0; a < nifx; ++a) on_x |= (ifx[a] - 1 == p);
      ry[u] = on_x ? make_double2(0, 0) : r[((int64_t)k * ny + ify[b] - 1) * nx + p];
    }
  }
}

__global__ void k_ml_lift(MlLift L, const double2* __restrict__ sig, const double2* __restrict__ f,
                          double2* __restrict__ f2) {
  const int64_t total = (int64_t)L.nz * L.nyc * L.nxc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(t % L.nxc);
    const int64_t rest = t / L.nxc;
    const int y = (int)(rest % L.nyc), k = (int)(rest / L.nyc);
    cplx acc = mk(0, 0);
    if (x == 0 && L.wL) acc = acc + mk(L.cL.x, L.cL.y) * ld(L.wL + k * L.ldx + L.ox + y);
    if (x == L.nxc - 1 && L.wR) acc = acc + mk(L.cR.x, L.cR.y) * ld(L.wR + k * L.ldx + L.ox + y);
    if (y == 0 && L.wB) acc = acc + mk(L.cB.x, L.cB.y) * ld(L.wB + k * L.ldy + L.oy + x);
    if (y == L.nyc - 1 && L.wT) acc = acc + mk(L.cT.x, L.cT.y) * ld(L.wT + k * L.ldy + L.oy + x);
    const cplx v = ld(f + t) - ld(sig + k) * acc;
    f2[t] = make_double2(v.x, v.y);
  }
}

cudaError_t launch_ml_gather(const double2* r, int nx, int ny, int nz, const int* d_ifx, int nifx, const int* d_ify,
                             int nify, double2* rx, double2* ry, cudaStream_t st) {
  const int64_t total = (int64_t)nifx * nz * ny + (int64_t)nify * nz * nx;
  if (!total) return cudaSuccess;
  k_ml_gather<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(r, nx, ny, nz, d_ifx, nifx,
                                                                                            d_ify, nify, rx, ry);
  return cudaGetLastError();
}
cudaError_t launch_ml_lift(const MlLift& L, const double2* sig, const double2* f, double2* f2, cudaStream_t st) {
  const int64_t total = (int64_t)L.nz * L.nyc * L.nxc;
  if (!total) return cudaSuccess;
  k_ml_lift<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(L, sig, f, f2);
  return cudaGetLastError();
}

}  // namespace lfds
