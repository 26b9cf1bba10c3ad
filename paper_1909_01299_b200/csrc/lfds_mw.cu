// Lebedev-grid Maxwell solve in a horizontally layered medium — PAPER.md §3 (lines 81-372).
//
//   A_h H = curl_h(rho curl_h H) - i omega mu H = f       (Eq. (abstr), (fin))
//
// on the grid M (N = 2n + 1 nodes per axis, 0-based, both ends primary: reading M1 of DESIGN.md
// §13), H (3 components) on the interior P nodes (i + j + k even), rho = diag(c1, c2, c3)(z) on
// the R nodes, boundary conditions H x n = 0 on dOmega ∩ P and E x n = 0 on dOmega ∩ R
// (PAPER.md:238-241).  The solve is the paper's separable route:
//
//  1. gather      the four Lebedev families of each level into packed arrays (k_mw_gather):
//                 pp, dd on even levels, pd, dp on odd levels;
//  2. transforms  along x and y in the family's 1D eigenbasis — primary axes Dirichlet, dual
//                 axes Neumann ("Dirichlet conditions on primary grid and Neumann conditions on
//                 dual grid"), the dual basis derived from the primary one
//                 (phi^d = phi^p_x / lambda, reading M4) — on the FP64 tensor pipe (the DMMA
//                 k_xform / k_xform3m of the scalar solver, lfds_xform.cu);
//  3. per harmonic (l, m) four decoupled systems (reading M5: {H^pp_x, H^dd_y, H^dp_z},
//                 {H^dd_x, H^pp_y, H^pd_z}, {H^pd_x, H^dp_y, H^dd_z}, {H^dp_x, H^pd_y, H^pp_z});
//                 H_z is eliminated by the third equation of each set ("each H_z may be expressed
//                 in terms of H_x and H_y"), leaving a block-tridiagonal system
//                 with 2x2 blocks along z, solved by block Thomas, one thread
//                 per (system, l, m) (k_mw_zsolve), H_z recovered in the backward sweep;
//  4. inverse transforms and scatter (k_mw_scatter).
// lfds_mw_residual evaluates r = f - A_h H directly on the grid (k_mw_curlh, k_mw_curle).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lfds.h"
#include "lfds_eig.h"
#include "lfds_internal.h"

namespace {

using zc = std::complex<double>;
thread_local std::string g_mw_err;

int mwfail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_mw_err = buf;
  return code;
}
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------- device complex helpers
struct cx {
  double x, y;
};
__device__ __forceinline__ cx mk(double a, double b) { return cx{a, b}; }
__device__ __forceinline__ cx ld(const double2* p) {
  const double2 v = __ldg(p);
  return cx{v.x, v.y};
}
__device__ __forceinline__ cx ldw(const double2* p) {  // (written by this kernel: no __ldg)
  const double2 v = *p;
  return cx{v.x, v.y};
}
__device__ __forceinline__ void st(double2* p, cx v) { *p = make_double2(v.x, v.y); }
__device__ __forceinline__ cx operator+(cx a, cx b) { return cx{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cx operator-(cx a, cx b) { return cx{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cx operator-(cx a) { return cx{-a.x, -a.y}; }
__device__ __forceinline__ cx operator*(cx a, cx b) { return cx{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cx cinv(cx a) {
  // one division: |a|^2 of the z-system entries stays far inside the double range
  const double r = 1.0 / fma(a.x, a.x, a.y * a.y);
  return cx{a.x * r, -a.y * r};
}
struct m2 {  // 2x2 complex matrix [[a, b], [c, d]]
  cx a, b, c, d;
};
struct v2 {
  cx x, y;
};
__device__ __forceinline__ m2 mmul(const m2& p, const m2& q) {
  return m2{p.a * q.a + p.b * q.c, p.a * q.b + p.b * q.d, p.c * q.a + p.d * q.c, p.c * q.b + p.d * q.d};
}
__device__ __forceinline__ v2 mvec(const m2& p, const v2& v) { return v2{p.a * v.x + p.b * v.y, p.c * v.x + p.d * v.y}; }
__device__ __forceinline__ m2 msub(const m2& p, const m2& q) { return m2{p.a - q.a, p.b - q.b, p.c - q.c, p.d - q.d}; }
__device__ __forceinline__ v2 vsub(const v2& p, const v2& q) { return v2{p.x - q.x, p.y - q.y}; }
__device__ __forceinline__ m2 minv(const m2& p) {
  const cx r = cinv(p.a * p.d - p.b * p.c);
  return m2{p.d * r, -(p.b * r), -(p.c * r), p.a * r};
}

// Family order and the four systems (reading M5).  kind: 0 = primary, 1 = dual.
//   family f: pp = 0, dd = 1, pd = 2, dp = 3; x-kind / y-kind; level parity (0 = even levels)
__host__ __device__ __forceinline__ int fam_xk(int f) { return f == 1 || f == 3; }
__host__ __device__ __forceinline__ int fam_yk(int f) { return f == 1 || f == 2; }
__host__ __device__ __forceinline__ int fam_of(int xk, int yk) { return xk == yk ? xk : (xk == 0 ? 2 : 3); }
// system s: the H_z family (a, b); H_x is (1-a, b), H_y is (a, 1-b)
__host__ __device__ __forceinline__ int sys_a(int s) { return s == 0 || s == 2; }  // A: dp, A': pd, C: dd, D: pp
__host__ __device__ __forceinline__ int sys_b(int s) { return s == 1 || s == 2; }

struct MwDev {
  int Nx, Ny, Nz, nx, ny, nz;
  int64_t fam_off[4];  // offsets (complex) of the families in a FAM-layout array
  int nlev[4];
  int64_t plane;       // ny * nx
  const double2* lam;  // nx (lambda_l, lambda_0 = 0)
  const double2* nu;   // ny
  const double2* lev;  // per level k: [dz_k, c1, c2, c3] (4 Nz)
  const double2* idz;  // 1 / dz_k (Nz)
  const double2* dxx;  // x_{i+1} - x_{i-1} per node (Nx), dyy (Ny), dzz (Nz)
  const double2* dyy;
  const double2* dzz;
  double2 iwm;         // i omega mu
};

__device__ __forceinline__ int lev_of(int f, int k) { return f < 2 ? (k >> 1) - 1 : (k - 1) >> 1; }

// ---------------------------------------------------------------- gather / scatter
// One row (component c, level k, y index j) of the field per CTA iteration: the row's family,
// packed y index and destination row are fixed (the P nodes of a row have i = j + k mod 2), so
// the element loop carries no index divisions.
__global__ void k_mw_gather(MwDev D, const double2* __restrict__ F, double2* __restrict__ fam) {
  const int64_t rows = (int64_t)3 * D.Nz * D.Ny;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int j = (int)(row % D.Ny);
    const int64_t rk = row / D.Ny;
    const int k = (int)(rk % D.Nz), c = (int)(rk / D.Nz);
    if (j == 0 || k == 0 || j == D.Ny - 1 || k == D.Nz - 1) continue;  // uniform over the CTA
    const int xk = (j + k) & 1, yk = j & 1, f = fam_of(xk, yk);
    const int yy = yk ? (j - 1) >> 1 : (j >> 1) - 1;
    double2* dst = fam + D.fam_off[f] + (((int64_t)c * D.nlev[f] + lev_of(f, k)) * D.ny + yy) * D.nx;
    const double2* src = F + row * D.Nx;
    for (int q = threadIdx.x;; q += blockDim.x) {  // i = 2q + xk, interior i in [1, Nx - 2]
      const int i = 2 * q + xk;
      if (i > D.Nx - 2) break;
      if (i > 0) dst[xk ? q : q - 1] = src[i];
    }
  }
}

__global__ void k_mw_scatter(MwDev D, const double2* __restrict__ fam, double2* __restrict__ H) {
  const int64_t rows = (int64_t)3 * D.Nz * D.Ny;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int j = (int)(row % D.Ny);
    const int64_t rk = row / D.Ny;
    const int k = (int)(rk % D.Nz), c = (int)(rk / D.Nz);
    const bool rok = j > 0 && k > 0 && j < D.Ny - 1 && k < D.Nz - 1;
    const int xk = (j + k) & 1, yk = j & 1, f = fam_of(xk, yk);
    const int yy = yk ? (j - 1) >> 1 : (j >> 1) - 1;
    const double2* src =
        rok ? fam + D.fam_off[f] + (((int64_t)c * D.nlev[f] + lev_of(f, k)) * D.ny + yy) * D.nx : fam;
    double2* dst = H + row * D.Nx;
    for (int i = threadIdx.x; i < D.Nx; i += blockDim.x) {
      double2 v = make_double2(0, 0);
      if (rok && (i & 1) == xk && i > 0 && i < D.Nx - 1) v = src[xk ? (i - 1) >> 1 : (i >> 1) - 1];
      dst[i] = v;
    }
  }
}

// ---------------------------------------------------------------- per-harmonic z-systems
// One thread per (system s, m, l).  With sx = s_x(a) (+lambda_l primary, -lambda_l dual),
// sy = s_y(b) and delta_k = c2 sx^2 + c1 sy^2 - i w mu at a level k of H_z:
//   H_z(k) = (f_z + sx c2 Dz H_x + sy c1 Dz H_y) / delta            (third equation)
//   G(k) = [E_y; E_x] = Q(k) Dz X(k) + q(k) f_z(k),  X = [H_x; H_y]  (E at the H_z levels)
//   rows at the X levels k:  S (G(k+1) - G(k-1)) / dz_k + C3(k) X(k) - i w mu X(k) = f_xy(k)
// with S = diag(-1, 1), S Q = (1/delta)[[-c2(c1 sy^2 - iwm), c1 c2 sx sy], [c1 c2 sx sy,
// -c1(c2 sx^2 - iwm)]], S q = (1/delta)[c2 sx; c1 sy], C3 = c3 [[sy^2, -sx sy], [-sx sy, sx^2]].
// G vanishes on the boundary levels (tangential E) and X on them (H on dOmega ∩ P).
struct Lev {
  m2 SQ;
  cx sqx, sqy, idel, c1, c2;
};
__device__ __forceinline__ Lev level_terms(const MwDev& D, int k, cx sx, cx sy) {
  const cx c1 = ld(D.lev + 4 * k + 1), c2 = ld(D.lev + 4 * k + 2);
  const cx iwm = mk(D.iwm.x, D.iwm.y);
  const cx sx2 = sx * sx, sy2 = sy * sy, sxy = sx * sy;
  const cx idel = cinv(c2 * sx2 + c1 * sy2 - iwm);
  Lev L;
  L.idel = idel;
  L.c1 = c1;
  L.c2 = c2;
  const cx c12 = c1 * c2 * sxy * idel;
  L.SQ = m2{-(c2 * (c1 * sy2 - iwm) * idel), c12, c12, -(c1 * (c2 * sx2 - iwm) * idel)};
  L.sqx = c2 * sx * idel;
  L.sqy = c1 * sy * idel;
  return L;
}

// fam2 (optional, the two-level step 5): a second right-hand-side array in the same layout,
// added to fam's on reading (the x-plane and y-plane parts of the transformed residual).
// (128, 3): 164 registers, no spills with the one-row-ahead loads (2.15 ms at the
// 128-register cap of 4 CTAs per SM, 2.00 ms here)
template <bool SUM>  // SUM: fam2 given (its values added on reading)
__global__ void __launch_bounds__(128, 3) k_mw_zsolve(MwDev D, double2* __restrict__ fam, double2* __restrict__ cp,
                                                   const double2* __restrict__ fam2) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)4 * D.plane) return;
  const int l = (int)(t % D.nx), m = (int)((t / D.nx) % D.ny), s = (int)(t / D.plane);
  const int a = sys_a(s), b = sys_b(s);
  const int fz = fam_of(a, b), fx = fam_of(1 - a, b), fy = fam_of(a, 1 - b);
  const cx lam = ld(D.lam + l), nu = ld(D.nu + m);
  const cx sx = a == 0 ? lam : -lam, sy = b == 0 ? nu : -nu;
  auto absent = [&](int f) { return (fam_xk(f) == 0 && l == 0) || (fam_yk(f) == 0 && m == 0); };
  const bool ax = absent(fx), ay = absent(fy), az = absent(fz);
  const int64_t hoff = (int64_t)m * D.nx + l;
  // X levels: even interior for s = 0, 1 (pp/dd in-plane), odd for s = 2, 3
  const int k0 = s < 2 ? 2 : 1, nX = s < 2 ? D.nz - 1 : D.nz;
  double2* FX = fam + D.fam_off[fx] + hoff;                                  // comp 0
  double2* FY = fam + D.fam_off[fy] + (int64_t)D.nlev[fy] * D.plane + hoff;  // comp 1
  double2* FZ = fam + D.fam_off[fz] + (int64_t)2 * D.nlev[fz] * D.plane + hoff;
  double2* CP = cp + (int64_t)s * (D.nz) * 4 * D.plane + hoff;
  const cx zero = mk(0, 0);
  const cx iwm = mk(D.iwm.x, D.iwm.y);
  const int64_t d2 = SUM ? (int64_t)(fam2 - fam) : 0;  // element offset of the second array
  auto rd = [&](const double2* p) -> cx { return SUM ? ldw(p) + ldw(p + d2) : ldw(p); };
  auto interior = [&](int k) { return k >= 1 && k <= D.Nz - 2; };
  // The volume loads of row r + 1 are issued before row r is eliminated (raw values: with fam2
  // the two parts are summed at use), so each row's memory latency overlaps the previous row's
  // arithmetic instead of serialising the sweep.
  struct Raw {
    cx x, y, z, x2, y2, z2;
  };
  auto fetch = [&](int k, Raw& v) {  // f_x, f_y at the X level k, f_z at k + 1
    const double2* px = FX + (int64_t)lev_of(fx, k) * D.plane;
    const double2* py = FY + (int64_t)lev_of(fy, k) * D.plane;
    const bool hz = !az && interior(k + 1);
    const double2* pz = FZ + (int64_t)lev_of(fz, k + 1) * D.plane;
    v.x = ax ? zero : ldw(px);
    v.y = ay ? zero : ldw(py);
    v.z = hz ? ldw(pz) : zero;
    if (SUM) {
      v.x2 = ax ? zero : ldw(px + d2);
      v.y2 = ay ? zero : ldw(py + d2);
      v.z2 = hz ? ldw(pz + d2) : zero;
    } else {
      v.x2 = v.y2 = v.z2 = zero;
    }
  };
  // forward sweep
  Lev Lm{};
  bool gm = interior(k0 - 1);
  if (gm) Lm = level_terms(D, k0 - 1, sx, sy);
  cx fzm = gm && !az ? rd(FZ + (int64_t)lev_of(fz, k0 - 1) * D.plane) : zero;
  m2 Cprev{};
  v2 Yprev{};
  Raw nx_;
  fetch(k0, nx_);
  for (int r = 0; r < nX; ++r) {
    const int k = k0 + 2 * r;
    const Raw cur = nx_;
    if (r + 1 < nX) fetch(k + 2, nx_);
    const cx idz = ld(D.idz + k);
    const bool gp = interior(k + 1);
    Lev Lp{};
    cx fzp = zero;
    if (gp) {
      Lp = level_terms(D, k + 1, sx, sy);
      fzp = cur.z + cur.z2;
    }
    m2 Ap{zero, zero, zero, zero}, Am{zero, zero, zero, zero};
    if (gp) {
      const cx w = idz * ld(D.idz + k + 1);
      Ap = m2{Lp.SQ.a * w, Lp.SQ.b * w, Lp.SQ.c * w, Lp.SQ.d * w};
    }
    if (gm) {
      const cx w = idz * ld(D.idz + k - 1);
      Am = m2{Lm.SQ.a * w, Lm.SQ.b * w, Lm.SQ.c * w, Lm.SQ.d * w};
    }
    const cx c3 = ld(D.lev + 4 * k + 3);
    m2 Dg{c3 * sy * sy - iwm, -(c3 * sx * sy), -(c3 * sx * sy), c3 * sx * sx - iwm};
    Dg = msub(msub(Dg, Ap), Am);
    const int lx = lev_of(fx, k), ly = lev_of(fy, k);
    v2 rhs{cur.x + cur.x2, cur.y + cur.y2};
    if (gp) rhs = vsub(rhs, v2{Lp.sqx * fzp * idz, Lp.sqy * fzp * idz});
    if (gm) rhs = v2{rhs.x + Lm.sqx * fzm * idz, rhs.y + Lm.sqy * fzm * idz};
    if (r > 0) {
      Dg = msub(Dg, mmul(Am, Cprev));
      rhs = vsub(rhs, mvec(Am, Yprev));
    }
    const m2 Di = minv(Dg);
    Cprev = mmul(Di, Ap);
    Yprev = mvec(Di, rhs);
    st(CP, Cprev.a);
    st(CP + D.plane, Cprev.b);
    st(CP + 2 * D.plane, Cprev.c);
    st(CP + 3 * D.plane, Cprev.d);
    CP += 4 * D.plane;
    st(FX + (int64_t)lx * D.plane, Yprev.x);
    st(FY + (int64_t)ly * D.plane, Yprev.y);
    Lm = Lp;
    gm = gp;
    fzm = fzp;
  }
  // backward sweep, H_z at the level between X(k) and X(k + 2) (and below the first X level)
  auto hz_at = [&](int kz, v2 Xlo, v2 Xhi, cx fzv) {  // X at kz - 1, kz + 1; fzv = f_z(kz)
    const Lev L = level_terms(D, kz, sx, sy);
    const cx idz = ld(D.idz + kz);
    const cx dzx = (Xhi.x - Xlo.x) * idz, dzy = (Xhi.y - Xlo.y) * idz;
    const cx v = (fzv + sx * L.c2 * dzx + sy * L.c1 * dzy) * L.idel;
    st(FZ + (int64_t)lev_of(fz, kz) * D.plane, az ? zero : v);
  };
  auto rdz = [&](int k) -> cx { return az ? zero : rd(FZ + (int64_t)lev_of(fz, k) * D.plane); };
  v2 Xn = Yprev;  // X at the last X level
  {
    const int k = k0 + 2 * (nX - 1);
    st(FX + (int64_t)lev_of(fx, k) * D.plane, ax ? zero : Xn.x);
    st(FY + (int64_t)lev_of(fy, k) * D.plane, ay ? zero : Xn.y);
    if (interior(k + 1)) hz_at(k + 1, Xn, v2{zero, zero}, rdz(k + 1));
  }
  CP -= 4 * D.plane;  // (row nX - 1's C' multiplies nothing)
  // row r of the backward sweep reads C'(r), Y(r) and f_z(k + 1); those of row r - 1 are in flight
  struct Back {
    m2 C;
    v2 Y;
    cx z, z2;
  };
  auto fetchb = [&](int r, const double2* cpr, Back& v) {
    const int k = k0 + 2 * r;
    v.C = m2{ldw(cpr), ldw(cpr + D.plane), ldw(cpr + 2 * D.plane), ldw(cpr + 3 * D.plane)};
    v.Y = v2{ldw(FX + (int64_t)lev_of(fx, k) * D.plane), ldw(FY + (int64_t)lev_of(fy, k) * D.plane)};
    const double2* pz = FZ + (int64_t)lev_of(fz, k + 1) * D.plane;
    v.z = az ? zero : ldw(pz);
    v.z2 = (az || !SUM) ? zero : ldw(pz + d2);
  };
  Back nb;
  if (nX >= 2) fetchb(nX - 2, CP - 4 * D.plane, nb);
  for (int r = nX - 2; r >= 0; --r) {
    const int k = k0 + 2 * r;
    CP -= 4 * D.plane;
    const Back cb = nb;
    if (r > 0) fetchb(r - 1, CP - 4 * D.plane, nb);
    const int lx = lev_of(fx, k), ly = lev_of(fy, k);
    const v2 X = vsub(cb.Y, mvec(cb.C, Xn));
    st(FX + (int64_t)lx * D.plane, ax ? zero : X.x);
    st(FY + (int64_t)ly * D.plane, ay ? zero : X.y);
    hz_at(k + 1, X, Xn, cb.z + cb.z2);
    Xn = X;
  }
  if (interior(k0 - 1)) hz_at(k0 - 1, v2{zero, zero}, Xn, rdz(k0 - 1));
}

void mw_zsolve_launch(const MwDev& D, double2* fam, double2* cp, const double2* fam2, cudaStream_t st) {
  const unsigned grid = (unsigned)((4 * D.plane + 127) / 128);
  if (fam2) k_mw_zsolve<true><<<grid, 128, 0, st>>>(D, fam, cp, fam2);
  else k_mw_zsolve<false><<<grid, 128, 0, st>>>(D, fam, cp, nullptr);
}

// ---------------------------------------------------------------- residual r = f - A_h H
// E = rho curl_h H on the interior R nodes (0 elsewhere), then r = f - (curl_h E - i w mu H)
// on the interior P nodes (0 elsewhere): Eq. (fin) / (abstr) evaluated directly.
__global__ void k_mw_curlh(MwDev D, const double2* __restrict__ H, double2* __restrict__ E) {
  const int64_t N = (int64_t)D.Nz * D.Ny * D.Nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % D.Nx);
    const int j = (int)((t / D.Nx) % D.Ny), k = (int)(t / ((int64_t)D.Nx * D.Ny));
    cx ex = mk(0, 0), ey = ex, ez = ex;
    if (((i + j + k) & 1) && i > 0 && j > 0 && k > 0 && i < D.Nx - 1 && j < D.Ny - 1 && k < D.Nz - 1) {
      const int64_t sx = 1, sy = D.Nx, sz = (int64_t)D.Nx * D.Ny;
      const cx ix = cinv(ld(D.dxx + i)), iy = cinv(ld(D.dyy + j)), iz = cinv(ld(D.dzz + k));
      // H enters only on the interior P nodes (Pi_P of the oracle): a neighbour on dOmega reads 0
      const bool xlo = i > 1, xhi = i < D.Nx - 2, ylo = j > 1, yhi = j < D.Ny - 2, zlo = k > 1, zhi = k < D.Nz - 2;
      auto d = [&](int c, int64_t s, bool lo, bool hi, cx inv) {
        const cx a = hi ? ld(H + c * N + t + s) : mk(0, 0), b = lo ? ld(H + c * N + t - s) : mk(0, 0);
        return (a - b) * inv;
      };
      ex = ld(D.lev + 4 * k + 1) * (d(2, sy, ylo, yhi, iy) - d(1, sz, zlo, zhi, iz));
      ey = ld(D.lev + 4 * k + 2) * (d(0, sz, zlo, zhi, iz) - d(2, sx, xlo, xhi, ix));
      ez = ld(D.lev + 4 * k + 3) * (d(1, sx, xlo, xhi, ix) - d(0, sy, ylo, yhi, iy));
    }
    st(E + t, ex);
    st(E + N + t, ey);
    st(E + 2 * N + t, ez);
  }
}

__global__ void k_mw_curle(MwDev D, const double2* __restrict__ E, const double2* __restrict__ H,
                           const double2* __restrict__ F, double2* __restrict__ R) {
  const int64_t N = (int64_t)D.Nz * D.Ny * D.Nx;
  const cx iwm = mk(D.iwm.x, D.iwm.y);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % D.Nx);
    const int j = (int)((t / D.Nx) % D.Ny), k = (int)(t / ((int64_t)D.Nx * D.Ny));
    cx rx = mk(0, 0), ry = rx, rz = rx;
    if (!((i + j + k) & 1) && i > 0 && j > 0 && k > 0 && i < D.Nx - 1 && j < D.Ny - 1 && k < D.Nz - 1) {
      const int64_t sx = 1, sy = D.Nx, sz = (int64_t)D.Nx * D.Ny;
      const cx ix = cinv(ld(D.dxx + i)), iy = cinv(ld(D.dyy + j)), iz = cinv(ld(D.dzz + k));
      auto d = [&](int c, int64_t s, cx inv) { return (ld(E + c * N + t + s) - ld(E + c * N + t - s)) * inv; };
      rx = ld(F + t) - (d(2, sy, iy) - d(1, sz, iz) - iwm * ld(H + t));
      ry = ld(F + N + t) - (d(0, sz, iz) - d(2, sx, ix) - iwm * ld(H + N + t));
      rz = ld(F + 2 * N + t) - (d(1, sx, ix) - d(0, sy, iy) - iwm * ld(H + 2 * N + t));
    }
    st(R + t, rx);
    st(R + N + t, ry);
    st(R + 2 * N + t, rz);
  }
}

enum { MK_GATHER = 0, MK_XF, MK_YF, MK_Z, MK_YI, MK_XI, MK_SCATTER, MK_N };
const char* const kMwNames[MK_N] = {"k_mw_gather", "k_mw_xfwd", "k_mw_yfwd", "k_mw_zsolve",
                                    "k_mw_yinv",   "k_mw_xinv", "k_mw_scatter"};

}  // namespace

struct lfds_mw {
  MwDev D{};
  int device = 0;
  bool realx = true, realy = true;
  char* d_mem = nullptr;         // TAB (transform matrices) + lam, nu, lev, dxx, dyy, dzz
  lfds::GemmDesc* d_desc = nullptr;  // [xf 4][yf 4][yi 4][xi 4]
  int maxMx = 0, maxMy = 0;
  int64_t maxNx = 0, maxNy = 0;
  size_t fam_elems = 0, cp_elems = 0;
  int profile = 0;
  cudaEvent_t ev[MK_N + 1] = {};
  double ms[MK_N] = {};
  int launches[MK_N] = {};
  bool ev_pending = false;
};

namespace {

// 1D bases of one axis: primary (Dirichlet) pencil S_p phi = lambda^2 D_p phi on the n - 1
// interior primary nodes (steps D_d between consecutive primary nodes, mass D_p = distance of the
// two dual neighbours), dual basis psi_l = (phi_l(b) - phi_l(b-1)) / (D_d(b) lambda_l) plus the
// Neumann null mode psi_0 = 1 / sqrt(sum D_d) (reading M4).  Forward matrices W^T diag(mass),
// inverse W; row-major [mode][node] and [node][mode].
struct Axis1 {
  int n = 0;
  bool real = true;
  std::vector<zc> lam;                 // n: lambda_0 = 0, lambda_l (l >= 1)
  std::vector<zc> Fp, Ip, Fd, Id;      // (n-1)x(n-1), (n-1)x(n-1), n x n, n x n
  std::vector<zc> dnode;               // x_{i+1} - x_{i-1} per node (1 at the ends)
};

int axis_setup(int N, const lfds_z* h, const char* name, Axis1& A) {
  if (N < 5 || !(N & 1)) return mwfail(LFDS_EINVAL, "%s: node count %d must be odd and >= 5", name, N);
  const int n = (N - 1) / 2;
  A.n = n;
  std::vector<zc> x(N);
  x[0] = 0;
  for (int t = 0; t + 1 < N; ++t) {
    x[t + 1] = x[t] + zc(h[t].re, h[t].im);
    if (h[t].im != 0) A.real = false;
    if (h[t].re == 0 && h[t].im == 0) return mwfail(LFDS_EINVAL, "%s: zero step %d", name, t);
  }
  A.dnode.assign(N, zc(1));
  for (int i = 1; i + 1 < N; ++i) A.dnode[i] = x[i + 1] - x[i - 1];
  std::vector<zc> Dd(n), Dp(n - 1);
  for (int b = 1; b <= n; ++b) Dd[b - 1] = x[2 * b] - x[2 * b - 2];
  for (int a = 1; a < n; ++a) Dp[a - 1] = x[2 * a + 1] - x[2 * a - 1];
  lfds::Basis B;
  std::string err;
  if (!lfds::pencil_basis(Dd, B, err, &Dp)) return mwfail(LFDS_EEIG, "%s primary pencil: %s", name, err.c_str());
  if (B.residual > 1e-10 || B.biorth > 1e-8)
    return mwfail(LFDS_EEIG, "%s primary basis inaccurate (residual %.2e, biorth %.2e)", name, B.residual, B.biorth);
  const int np = n - 1;
  A.lam.assign(n, zc(0));
  for (int c = 0; c < np; ++c) {
    A.lam[c + 1] = std::sqrt(-B.lam[c]);
    if (std::abs(A.lam[c + 1]) == 0) return mwfail(LFDS_ERESONANCE, "%s: zero primary eigenvalue", name);
  }
  A.Fp.assign((size_t)np * np, 0);
  A.Ip.assign((size_t)np * np, 0);
  for (int a = 0; a < np; ++a)
    for (int c = 0; c < np; ++c) {
      const zc w = B.W[(size_t)a * np + c];
      A.Ip[(size_t)a * np + c] = w;        // [node a][mode c + 1]
      A.Fp[(size_t)c * np + a] = w * Dp[a];  // [mode c + 1][node a]
    }
  A.Fd.assign((size_t)n * n, 0);
  A.Id.assign((size_t)n * n, 0);
  zc sum = 0;
  for (int b = 0; b < n; ++b) sum += Dd[b];
  const zc psi0 = 1.0 / std::sqrt(sum);
  for (int b = 0; b < n; ++b) {  // dual node b + 1 (i = 2b + 1) sits between primary a = b and b + 1
    for (int l = 0; l < n; ++l) {
      zc psi;
      if (l == 0) {
        psi = psi0;
      } else {
        const zc hi = b + 1 <= np ? B.W[(size_t)b * np + (l - 1)] : zc(0);   // phi at primary b + 1
        const zc lo = b >= 1 ? B.W[(size_t)(b - 1) * np + (l - 1)] : zc(0);   // phi at primary b
        psi = (hi - lo) / (Dd[b] * A.lam[l]);
      }
      A.Id[(size_t)b * n + l] = psi;
      A.Fd[(size_t)l * n + b] = psi * Dd[b];
    }
  }
  return LFDS_OK;
}

}  // namespace

extern "C" {

const char* lfds_mw_last_error(void) { return g_mw_err.c_str(); }
int lfds_mw_kernel_count(void) { return MK_N; }
const char* lfds_mw_kernel_name(int k) { return k >= 0 && k < MK_N ? kMwNames[k] : ""; }

void lfds_mw_destroy(lfds_mw* P) {
  if (!P) return;
  cudaFree(P->d_mem);
  cudaFree(P->d_desc);
  for (auto& e : P->ev)
    if (e) cudaEventDestroy(e);
  delete P;
}

int lfds_mw_setup(int Nx, const lfds_z* hx, int Ny, const lfds_z* hy, int Nz, const lfds_z* hz, const lfds_z* c1,
                  const lfds_z* c2, const lfds_z* c3, lfds_z mu, double omega, int device, int profile,
                  lfds_mw** out) {
  if (!out || !hx || !hy || !hz || !c1 || !c2 || !c3) return mwfail(LFDS_EINVAL, "NULL argument");
  *out = nullptr;
  Axis1 X, Y, Z;
  int rc;
  if ((rc = axis_setup(Nx, hx, "x", X)) || (rc = axis_setup(Ny, hy, "y", Y)) || (rc = axis_setup(Nz, hz, "z", Z)))
    return rc;
  if (!(omega > 0)) return mwfail(LFDS_EINVAL, "omega must be > 0");
  if (cudaSetDevice(device) != cudaSuccess) return mwfail(LFDS_ENODEVICE, "no CUDA device %d", device);
  std::unique_ptr<lfds_mw> P(new lfds_mw());
  P->device = device;
  P->profile = profile;
  MwDev& D = P->D;
  D.Nx = Nx; D.Ny = Ny; D.Nz = Nz;
  D.nx = X.n; D.ny = Y.n; D.nz = Z.n;
  D.plane = (int64_t)D.nx * D.ny;
  D.nlev[0] = D.nlev[1] = D.nz - 1;
  D.nlev[2] = D.nlev[3] = D.nz;
  int64_t off = 0;
  for (int f = 0; f < 4; ++f) {
    D.fam_off[f] = off;
    off += (int64_t)3 * D.nlev[f] * D.plane;
  }
  P->fam_elems = (size_t)off;
  P->cp_elems = (size_t)4 * D.nz * 4 * D.plane;
  const zc iwm = zc(0, omega) * zc(mu.re, mu.im);
  D.iwm = make_double2(iwm.real(), iwm.imag());
  // per level: dz, c1, c2, c3; resonance of the H_z elimination
  std::vector<zc> lev(4 * (size_t)Nz);
  for (int k = 0; k < Nz; ++k) {
    lev[4 * k] = Z.dnode[k];
    lev[4 * k + 1] = zc(c1[k].re, c1[k].im);
    lev[4 * k + 2] = zc(c2[k].re, c2[k].im);
    lev[4 * k + 3] = zc(c3[k].re, c3[k].im);
  }
  {
    double worst = 1e300;
    int wl = 0, wm = 0, wk = 0;
    for (int k = 1; k + 1 < Nz; ++k)
      for (int l = 0; l < D.nx; ++l)
        for (int m = 0; m < D.ny; ++m) {
          const zc a = lev[4 * k + 2] * X.lam[l] * X.lam[l], b = lev[4 * k + 1] * Y.lam[m] * Y.lam[m];
          const double rel = std::abs(a + b - iwm) / (std::abs(a) + std::abs(b) + std::abs(iwm));
          if (rel < worst) { worst = rel; wl = l; wm = m; wk = k; }
        }
    if (worst < 1e-13)
      return mwfail(LFDS_ERESONANCE, "H_z elimination singular: harmonic (l, m) = (%d, %d), level %d (%.2e)", wl, wm,
                    wk, worst);
  }
  P->realx = X.real;
  P->realy = Y.real;
  // device memory: matrices then tables
  auto mat_bytes = [](const Axis1& A, size_t n2) { return al256(n2 * (A.real ? 8 : 16)); };
  const size_t npx = (size_t)(D.nx - 1) * (D.nx - 1), ndx = (size_t)D.nx * D.nx;
  const size_t npy = (size_t)(D.ny - 1) * (D.ny - 1), ndy = (size_t)D.ny * D.ny;
  size_t o = 0;
  const size_t oFpx = o; o += mat_bytes(X, npx);
  const size_t oIpx = o; o += mat_bytes(X, npx);
  const size_t oFdx = o; o += mat_bytes(X, ndx);
  const size_t oIdx = o; o += mat_bytes(X, ndx);
  const size_t oFpy = o; o += mat_bytes(Y, npy);
  const size_t oIpy = o; o += mat_bytes(Y, npy);
  const size_t oFdy = o; o += mat_bytes(Y, ndy);
  const size_t oIdy = o; o += mat_bytes(Y, ndy);
  const size_t oLam = o; o += al256(16 * (size_t)D.nx);
  const size_t oNu = o; o += al256(16 * (size_t)D.ny);
  const size_t oLev = o; o += al256(16 * lev.size());
  const size_t oDx = o; o += al256(16 * (size_t)Nx);
  const size_t oDy = o; o += al256(16 * (size_t)Ny);
  const size_t oDz = o; o += al256(16 * (size_t)Nz);
  const size_t oIdz = o; o += al256(16 * (size_t)Nz);
  std::vector<char> h(o, 0);
  auto put = [&](size_t at, const std::vector<zc>& v, bool real) {
    if (real) {
      double* d = reinterpret_cast<double*>(h.data() + at);
      for (size_t q = 0; q < v.size(); ++q) d[q] = v[q].real();
    } else {
      double2* d = reinterpret_cast<double2*>(h.data() + at);
      for (size_t q = 0; q < v.size(); ++q) d[q] = make_double2(v[q].real(), v[q].imag());
    }
  };
  put(oFpx, X.Fp, X.real); put(oIpx, X.Ip, X.real); put(oFdx, X.Fd, X.real); put(oIdx, X.Id, X.real);
  put(oFpy, Y.Fp, Y.real); put(oIpy, Y.Ip, Y.real); put(oFdy, Y.Fd, Y.real); put(oIdy, Y.Id, Y.real);
  put(oLam, X.lam, false); put(oNu, Y.lam, false); put(oLev, lev, false);
  put(oDx, X.dnode, false); put(oDy, Y.dnode, false); put(oDz, Z.dnode, false);
  {
    std::vector<zc> idz(Nz);
    for (int k = 0; k < Nz; ++k) idz[k] = 1.0 / Z.dnode[k];
    put(oIdz, idz, false);
  }
  if (cudaMalloc(&P->d_mem, o) != cudaSuccess) return mwfail(LFDS_ENOMEM, "device tables (%zu bytes)", o);
  if (cudaMemcpy(P->d_mem, h.data(), o, cudaMemcpyHostToDevice) != cudaSuccess)
    return mwfail(LFDS_ECUDA, "table upload");
  auto dp = [&](size_t at) { return reinterpret_cast<const double2*>(P->d_mem + at); };
  D.lam = dp(oLam); D.nu = dp(oNu); D.lev = dp(oLev); D.dxx = dp(oDx); D.dyy = dp(oDy); D.dzz = dp(oDz);
  D.idz = dp(oIdz);
  // transform descriptors (lfds_internal.h GemmDesc: C(i, n) = sum_j S(i, j) B(j, n)); the
  // buffers are B_MS = FAM (node data / coefficients) and B_T1 = T (half-transformed)
  std::vector<lfds::GemmDesc> desc;
  auto aoff = [](size_t byte_off, bool real) { return (int64_t)(byte_off / (real ? 8 : 16)); };
  const int64_t nx = D.nx, ny = D.ny, pl = D.plane;
  for (int pass = 0; pass < 4; ++pass) {  // 0 x-fwd, 1 y-fwd, 2 y-inv, 3 x-inv
    for (int f = 0; f < 4; ++f) {
      const int xk = fam_xk(f), yk = fam_yk(f);
      const int nxf = xk ? D.nx : D.nx - 1, nyf = yk ? D.ny : D.ny - 1;
      lfds::GemmDesc g{};
      g.N1 = 3 * D.nlev[f];
      g.sB1 = g.sC1 = pl;
      if (pass == 0) {
        g.a_off = aoff(xk ? oFdx : oFpx, X.real); g.sAi = nxf; g.sAj = 1; g.M = g.K = nxf;
        g.b_buf = lfds::B_MS; g.b_off = D.fam_off[f]; g.sBj = 1; g.N2 = nyf; g.sB2 = nx;
        g.c_buf = lfds::B_T1; g.c_off = D.fam_off[f] + (xk ? 0 : 1); g.sCi = 1; g.sC2 = nx;
      } else if (pass == 1) {
        g.a_off = aoff(yk ? oFdy : oFpy, Y.real); g.sAi = nyf; g.sAj = 1; g.M = g.K = nyf;
        g.b_buf = lfds::B_T1; g.b_off = D.fam_off[f]; g.sBj = nx; g.N2 = (int)nx; g.sB2 = 1;
        g.c_buf = lfds::B_MS; g.c_off = D.fam_off[f] + (yk ? 0 : nx); g.sCi = nx; g.sC2 = 1;
      } else if (pass == 2) {
        g.a_off = aoff(yk ? oIdy : oIpy, Y.real); g.sAi = nyf; g.sAj = 1; g.M = g.K = nyf;
        g.b_buf = lfds::B_MS; g.b_off = D.fam_off[f] + (yk ? 0 : nx); g.sBj = nx; g.N2 = (int)nx; g.sB2 = 1;
        g.c_buf = lfds::B_T1; g.c_off = D.fam_off[f]; g.sCi = nx; g.sC2 = 1;
      } else {
        g.a_off = aoff(xk ? oIdx : oIpx, X.real); g.sAi = nxf; g.sAj = 1; g.M = g.K = nxf;
        g.b_buf = lfds::B_T1; g.b_off = D.fam_off[f] + (xk ? 0 : 1); g.sBj = 1; g.N2 = nyf; g.sB2 = nx;
        g.c_buf = lfds::B_MS; g.c_off = D.fam_off[f]; g.sCi = 1; g.sC2 = nx;
      }
      desc.push_back(g);
      const int64_t N = (int64_t)g.N1 * g.N2;
      if (pass == 0 || pass == 3) { P->maxMx = std::max(P->maxMx, g.M); P->maxNx = std::max(P->maxNx, N); }
      else { P->maxMy = std::max(P->maxMy, g.M); P->maxNy = std::max(P->maxNy, N); }
    }
  }
  (void)ny;
  if (cudaMalloc(&P->d_desc, desc.size() * sizeof(lfds::GemmDesc)) != cudaSuccess ||
      cudaMemcpy(P->d_desc, desc.data(), desc.size() * sizeof(lfds::GemmDesc), cudaMemcpyHostToDevice) != cudaSuccess)
    return mwfail(LFDS_ECUDA, "descriptor upload");
  if (profile)
    for (auto& e : P->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return mwfail(LFDS_ECUDA, "event create");
  *out = P.release();
  return LFDS_OK;
}

size_t lfds_mw_workspace_bytes(const lfds_mw* P) {
  if (!P) return 0;
  const size_t solve = 2 * al256(P->fam_elems * 16) + al256(P->cp_elems * 16);
  const size_t resid = al256((size_t)3 * P->D.Nz * P->D.Ny * P->D.Nx * 16);
  return std::max(solve, resid);
}

int lfds_mw_solve(lfds_mw* P, const void* f_dev, void* h_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!P || !f_dev || !h_dev || !ws) return mwfail(LFDS_EINVAL, "bad arguments");
  if (ws_bytes < lfds_mw_workspace_bytes(P)) return mwfail(LFDS_EINVAL, "workspace too small");
  if (((uintptr_t)f_dev | (uintptr_t)h_dev | (uintptr_t)ws) & 15) return mwfail(LFDS_EINVAL, "pointers must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  (void)cudaGetLastError();
  char* w = static_cast<char*>(ws);
  double2* fam = reinterpret_cast<double2*>(w);
  double2* T = reinterpret_cast<double2*>(w + al256(P->fam_elems * 16));
  double2* cp = reinterpret_cast<double2*>(w + 2 * al256(P->fam_elems * 16));
  lfds::Bufs b{};
  b.p[lfds::B_TAB] = P->d_mem;
  b.p[lfds::B_MS] = fam;
  b.p[lfds::B_T1] = T;
  const unsigned gs = (unsigned)std::min<int64_t>((int64_t)3 * P->D.Nz * P->D.Ny, 148 * 16);  // rows
  cudaError_t e = cudaSuccess;
  auto mark = [&](int i) {
    if (P->profile) cudaEventRecord(P->ev[i], st);
  };
  mark(0);
  k_mw_gather<<<gs, 256, 0, st>>>(P->D, static_cast<const double2*>(f_dev), fam);
  mark(1);
  if (!e) e = cudaGetLastError();
  if (!e) e = lfds::launch_xform(P->d_desc + 0, 4, P->maxMx, P->maxNx, P->realx, true, b, st);
  mark(2);
  if (!e) e = lfds::launch_xform(P->d_desc + 4, 4, P->maxMy, P->maxNy, P->realy, false, b, st);
  mark(3);
  if (!e) {
    mw_zsolve_launch(P->D, fam, cp, nullptr, st);
    e = cudaGetLastError();
  }
  mark(4);
  if (!e) e = lfds::launch_xform(P->d_desc + 8, 4, P->maxMy, P->maxNy, P->realy, false, b, st);
  mark(5);
  if (!e) e = lfds::launch_xform(P->d_desc + 12, 4, P->maxMx, P->maxNx, P->realx, true, b, st);
  mark(6);
  if (!e) {
    k_mw_scatter<<<gs, 256, 0, st>>>(P->D, fam, static_cast<double2*>(h_dev));
    e = cudaGetLastError();
  }
  mark(7);
  if (e) return mwfail(LFDS_ECUDA, "maxwell solve: %s", cudaGetErrorString(e));
  if (P->profile) {
    // accumulate the previous solve's events (this solve's are read at the next call / query)
    P->ev_pending = true;
    cudaEventSynchronize(P->ev[MK_N]);
    for (int i = 0; i < MK_N; ++i) {
      float t = 0;
      cudaEventElapsedTime(&t, P->ev[i], P->ev[i + 1]);
      P->ms[i] += t;
      P->launches[i] += 1;
    }
    P->ev_pending = false;
  }
  return LFDS_OK;
}

int lfds_mw_kernel_times(lfds_mw* P, double* ms, int* launches) {
  if (!P) return mwfail(LFDS_EINVAL, "plan is NULL");
  for (int i = 0; i < MK_N; ++i) {
    if (ms) ms[i] = P->ms[i];
    if (launches) launches[i] = P->launches[i];
    P->ms[i] = 0;
    P->launches[i] = 0;
  }
  return LFDS_OK;
}

int lfds_mw_residual(lfds_mw* P, const void* h_dev, const void* f_dev, void* r_dev, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!P || !h_dev || !f_dev || !r_dev || !ws) return mwfail(LFDS_EINVAL, "bad arguments");
  if (ws_bytes < lfds_mw_workspace_bytes(P)) return mwfail(LFDS_EINVAL, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  (void)cudaGetLastError();
  const int64_t N = (int64_t)P->D.Nz * P->D.Ny * P->D.Nx;
  const unsigned gs = (unsigned)std::min<int64_t>((N + 255) / 256, 148 * 16);
  double2* E = static_cast<double2*>(ws);
  k_mw_curlh<<<gs, 256, 0, st>>>(P->D, static_cast<const double2*>(h_dev), E);
  k_mw_curle<<<gs, 256, 0, st>>>(P->D, E, static_cast<const double2*>(h_dev), static_cast<const double2*>(f_dev),
                                  static_cast<double2*>(r_dev));
  const cudaError_t e = cudaGetLastError();
  if (e) return mwfail(LFDS_ECUDA, "maxwell residual: %s", cudaGetErrorString(e));
  return LFDS_OK;
}

}  // extern "C"

// =====================================================================================
// Two-level (blocked) Maxwell solve: H = H^1 + H^2.
//
// The blocks S^ij lie between x-interfaces I_a and y-interfaces J_b (even nodes: every block is a
// Lebedev sub-grid whose boundary nodes are primary, reading M6).  With A_S the block operator
// (H x n = 0 on dS ∩ P, E x n = 0 on dS ∩ R — exactly the layered problem on the sub-grid):
//   1-3. v = H^1: A_S v_S = f_S on every block, v = 0 on the interface planes   (block plans)
//   4.   r = f - A_h v; it lives on the layers {I-1, I, I+1} x all y and all x x {J-1, J, J+1}
//        (the block equations next to a plane assumed E_tan = 0 on it; reading M6)
//   5.   w = A_h^{-1} r on those layers only ("computed on the fifth step"):
//        the global separable solve with its x- and y-transforms restricted to the layer
//        columns / rows — forward: y-transform of the K_x layer columns then the sparse x-sum,
//        x-transform of the K_y layer rows then the sparse y-sum; all harmonics' z-systems
//        (k_mw_zsolve with the two parts summed); inverse evaluated on the layers only;
//        H = v + w there, so H^2's boundary data are H_tan on the plane P nodes and
//        E_tan = (rho curl_h H)_tan on the plane R nodes ("imposed on both these grids")
//   6-7. A_S H_S = f_S - [curl_h E_b + curl_h (rho curl_h H_b)] next to dS (the interface data
//        lifted into the right side), block plans again; H = w on the plane P nodes.
// Exact like the scalar method: H = A_h^{-1} f up to rounding.
namespace {

__global__ void k_mw2_gather_r(MwDev D, const double2* __restrict__ r, double2* __restrict__ out,
                               const int64_t* __restrict__ cxo, const int64_t* __restrict__ cyo,
                               const int* __restrict__ lx, const int* __restrict__ ly, int Kx0, int Kx1, int Ky0,
                               int Ky1, const unsigned char* __restrict__ isx, int64_t total) {
  // compact layer arrays: x-part [f][c*lev][y-node][kx], y-part [f][c*lev][ky][x-node] (zero at
  // the x-layer columns, which the x-part carries)
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t;
    int part = 0, f = 0;
    int64_t sz = 0;
    for (part = 0; part < 2; ++part) {
      for (f = 0; f < 4; ++f) {
        const int K = part == 0 ? (fam_xk(f) ? Kx1 : Kx0) : (fam_yk(f) ? Ky1 : Ky0);
        sz = (int64_t)3 * D.nlev[f] * K * (part == 0 ? D.ny : D.nx);
        if (u < sz) break;
        u -= sz;
      }
      if (f < 4) break;
    }
    const int xk = fam_xk(f), yk = fam_yk(f);
    const int nxf = xk ? D.nx : D.nx - 1, nyf = yk ? D.ny : D.ny - 1;
    int i, j, cl;
    double2 v = make_double2(0, 0);
    bool ok;
    if (part == 0) {
      const int K = xk ? Kx1 : Kx0;
      const int kx = (int)(u % K);
      const int yy = (int)((u / K) % D.ny);
      cl = (int)(u / ((int64_t)K * D.ny));
      i = lx[xk * (Kx0 + 0) + kx];  // node of layer column kx (lists: primary then dual)
      j = yk ? 2 * yy + 1 : 2 * yy + 2;
      ok = yy < nyf;
    } else {
      const int K = yk ? Ky1 : Ky0;
      const int xx = (int)(u % D.nx);
      const int ky = (int)((u / D.nx) % K);
      cl = (int)(u / ((int64_t)K * D.nx));
      j = ly[yk * (Ky0 + 0) + ky];
      i = xk ? 2 * xx + 1 : 2 * xx + 2;
      ok = xx < nxf && !isx[i];
    }
    if (ok) {
      const int c = cl / D.nlev[f], lev = cl % D.nlev[f];
      const int k = f < 2 ? 2 * lev + 2 : 2 * lev + 1;
      v = r[(((int64_t)c * D.Nz + k) * D.Ny + j) * D.Nx + i];
    }
    out[(part == 0 ? cxo[f] : cyo[f]) + u] = v;
  }
}

__global__ void k_mw2_add_w(MwDev D, const double2* __restrict__ w, double2* __restrict__ H,
                            const int64_t* __restrict__ cxo, const int64_t* __restrict__ cyo,
                            const int* __restrict__ lx, const int* __restrict__ ly, int Kx0, int Kx1, int Ky0, int Ky1,
                            const unsigned char* __restrict__ isx, int64_t total) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t;
    int part = 0, f = 0;
    for (part = 0; part < 2; ++part) {
      for (f = 0; f < 4; ++f) {
        const int K = part == 0 ? (fam_xk(f) ? Kx1 : Kx0) : (fam_yk(f) ? Ky1 : Ky0);
        const int64_t sz = (int64_t)3 * D.nlev[f] * K * (part == 0 ? D.ny : D.nx);
        if (u < sz) break;
        u -= sz;
      }
      if (f < 4) break;
    }
    const int xk = fam_xk(f), yk = fam_yk(f);
    const int nxf = xk ? D.nx : D.nx - 1, nyf = yk ? D.ny : D.ny - 1;
    int i, j, cl;
    bool ok;
    if (part == 0) {
      const int K = xk ? Kx1 : Kx0;
      const int kx = (int)(u % K);
      const int yy = (int)((u / K) % D.ny);
      cl = (int)(u / ((int64_t)K * D.ny));
      i = lx[xk * Kx0 + kx];
      j = yk ? 2 * yy + 1 : 2 * yy + 2;
      ok = yy < nyf;
    } else {
      const int K = yk ? Ky1 : Ky0;
      const int xx = (int)(u % D.nx);
      const int ky = (int)((u / D.nx) % K);
      cl = (int)(u / ((int64_t)K * D.nx));
      j = ly[yk * Ky0 + ky];
      i = xk ? 2 * xx + 1 : 2 * xx + 2;
      ok = xx < nxf && !isx[i];
    }
    if (ok) {
      const int c = cl / D.nlev[f], lev = cl % D.nlev[f];
      const int k = f < 2 ? 2 * lev + 2 : 2 * lev + 1;
      const int64_t o = (((int64_t)c * D.Nz + k) * D.Ny + j) * D.Nx + i;
      const double2 a = H[o], b = w[(part == 0 ? cxo[f] : cyo[f]) + u];
      H[o] = make_double2(a.x + b.x, a.y + b.y);
    }
  }
}

// E_l on the interior R nodes: on an interface plane the true E = rho curl_h H (H = v + w on the
// layers), elsewhere rho curl_h H_b with H_b = H on the plane P nodes only (nonzero next to a
// plane).  Then f2 = f - curl_h E_l on the interior P nodes off the planes.
__global__ void k_mw2_elift(MwDev D, const double2* __restrict__ H, double2* __restrict__ E,
                            const unsigned char* __restrict__ plx, const unsigned char* __restrict__ ply) {
  const int64_t N = (int64_t)D.Nz * D.Ny * D.Nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % D.Nx);
    const int j = (int)((t / D.Nx) % D.Ny), k = (int)(t / ((int64_t)D.Nx * D.Ny));
    cx ex = mk(0, 0), ey = ex, ez = ex;
    if (((i + j + k) & 1) && i > 0 && j > 0 && k > 0 && i < D.Nx - 1 && j < D.Ny - 1 && k < D.Nz - 1) {
      const bool on = plx[i] || ply[j];
      const int64_t sx = 1, sy = D.Nx, sz = (int64_t)D.Nx * D.Ny;
      const cx ix = cinv(ld(D.dxx + i)), iy = cinv(ld(D.dyy + j)), iz = cinv(ld(D.dzz + k));
      // neighbour (di, dj, dk) is usable if interior and (on ? any : on a plane)
      auto use = [&](int ii, int jj, int kk) {
        if (ii <= 0 || jj <= 0 || kk <= 0 || ii >= D.Nx - 1 || jj >= D.Ny - 1 || kk >= D.Nz - 1) return false;
        return on || plx[ii] || ply[jj];
      };
      auto d = [&](int c, int di, int dj, int dk, int64_t s, cx inv) {
        const cx a = use(i + di, j + dj, k + dk) ? ld(H + c * N + t + s) : mk(0, 0);
        const cx b = use(i - di, j - dj, k - dk) ? ld(H + c * N + t - s) : mk(0, 0);
        return (a - b) * inv;
      };
      ex = ld(D.lev + 4 * k + 1) * (d(2, 0, 1, 0, sy, iy) - d(1, 0, 0, 1, sz, iz));
      ey = ld(D.lev + 4 * k + 2) * (d(0, 0, 0, 1, sz, iz) - d(2, 1, 0, 0, sx, ix));
      ez = ld(D.lev + 4 * k + 3) * (d(1, 1, 0, 0, sx, ix) - d(0, 0, 1, 0, sy, iy));
    }
    st(E + t, ex);
    st(E + N + t, ey);
    st(E + 2 * N + t, ez);
  }
}

__global__ void k_mw2_flift(MwDev D, const double2* __restrict__ E, const double2* __restrict__ F,
                            double2* __restrict__ F2, const unsigned char* __restrict__ plx,
                            const unsigned char* __restrict__ ply) {
  const int64_t N = (int64_t)D.Nz * D.Ny * D.Nx;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % D.Nx);
    const int j = (int)((t / D.Nx) % D.Ny), k = (int)(t / ((int64_t)D.Nx * D.Ny));
    cx rx = mk(0, 0), ry = rx, rz = rx;
    if (!((i + j + k) & 1) && i > 0 && j > 0 && k > 0 && i < D.Nx - 1 && j < D.Ny - 1 && k < D.Nz - 1 && !plx[i] &&
        !ply[j]) {
      const int64_t sx = 1, sy = D.Nx, sz = (int64_t)D.Nx * D.Ny;
      const cx ix = cinv(ld(D.dxx + i)), iy = cinv(ld(D.dyy + j)), iz = cinv(ld(D.dzz + k));
      auto d = [&](int c, int64_t s, cx inv) { return (ld(E + c * N + t + s) - ld(E + c * N + t - s)) * inv; };
      rx = ld(F + t) - (d(2, sy, iy) - d(1, sz, iz));
      ry = ld(F + N + t) - (d(0, sz, iz) - d(2, sx, ix));
      rz = ld(F + 2 * N + t) - (d(1, sx, ix) - d(0, sy, iy));
    }
    st(F2 + t, rx);
    st(F2 + N + t, ry);
    st(F2 + 2 * N + t, rz);
  }
}

}  // namespace

struct lfds_mw2 {
  lfds_mw* glob = nullptr;  // global grid: MwDev tables (lam, nu, levels, steps) and residual kernels
  struct Blk {
    lfds_mw* plan = nullptr;
    int x0, x1, y0, y1;  // box nodes (inclusive): its boundary nodes lie on planes / dOmega
  };
  std::vector<Blk> blk;
  bool realx = true, realy = true;
  char* d_tab = nullptr;            // step-5 matrices + layer tables
  lfds::GemmDesc* d_desc = nullptr;  // 8 groups of 4
  int Kx[2] = {0, 0}, Ky[2] = {0, 0};
  const int* d_lx = nullptr;
  const int* d_ly = nullptr;
  const unsigned char *d_isx = nullptr, *d_plx = nullptr, *d_ply = nullptr;
  const int64_t *d_cxo = nullptr, *d_cyo = nullptr;
  int64_t compact = 0;               // complex elements of one compact slot (>= 1)
  int64_t compact_used = 0;          // of which in use (0 without interfaces)
  int gM[8] = {}, gKc[8] = {}, gReal[8] = {};
  int64_t gN[8] = {};
  size_t sub_elems = 0, sub_ws = 0;
};

extern "C" {

void lfds_mw2_destroy(lfds_mw2* P) {
  if (!P) return;
  if (P->glob) lfds_mw_destroy(P->glob);
  for (auto& b : P->blk)
    if (b.plan) lfds_mw_destroy(b.plan);
  cudaFree(P->d_tab);
  cudaFree(P->d_desc);
  delete P;
}

int lfds_mw2_setup(int Nx, const lfds_z* hx, int Ny, const lfds_z* hy, int Nz, const lfds_z* hz, const lfds_z* c1,
                   const lfds_z* c2, const lfds_z* c3, lfds_z mu, double omega, int n_ix, const int* ix, int n_iy,
                   const int* iy, int device, lfds_mw2** out) {
  if (!out) return mwfail(LFDS_EINVAL, "out is NULL");
  *out = nullptr;
  auto check_if = [&](int N, int n, const int* I, const char* ax) -> int {
    int prev = 0;
    for (int a = 0; a < n; ++a) {
      if (I[a] % 2 || I[a] - prev < 4) return mwfail(LFDS_EINVAL, "%s interface %d: even nodes >= 4 apart", ax, I[a]);
      prev = I[a];
    }
    if (N - 1 - prev < 4) return mwfail(LFDS_EINVAL, "%s: last block narrower than 5 nodes", ax);
    return LFDS_OK;
  };
  int rc;
  if ((rc = check_if(Nx, n_ix, ix, "x")) || (rc = check_if(Ny, n_iy, iy, "y"))) return rc;
  std::unique_ptr<lfds_mw2> P(new lfds_mw2());
  auto bail = [&](int code) {
    lfds_mw2_destroy(P.release());
    return code;
  };
  if ((rc = lfds_mw_setup(Nx, hx, Ny, hy, Nz, hz, c1, c2, c3, mu, omega, device, 0, &P->glob))) return bail(rc);
  const MwDev& D = P->glob->D;
  // blocks and their plans (sub-grids of the steps)
  std::vector<int> xs = {0}, ys = {0};
  xs.insert(xs.end(), ix, ix + n_ix); xs.push_back(Nx - 1);
  ys.insert(ys.end(), iy, iy + n_iy); ys.push_back(Ny - 1);
  for (size_t b = 0; b + 1 < ys.size(); ++b)
    for (size_t a = 0; a + 1 < xs.size(); ++a) {
      lfds_mw2::Blk B{nullptr, xs[a], xs[a + 1], ys[b], ys[b + 1]};
      if ((rc = lfds_mw_setup(B.x1 - B.x0 + 1, hx + B.x0, B.y1 - B.y0 + 1, hy + B.y0, Nz, hz, c1, c2, c3, mu, omega,
                              device, 0, &B.plan))) {
        P->blk.push_back(B);
        return bail(rc);
      }
      P->blk.push_back(B);
      P->sub_elems = std::max(P->sub_elems, (size_t)3 * Nz * (B.y1 - B.y0 + 1) * (B.x1 - B.x0 + 1));
      P->sub_ws = std::max(P->sub_ws, lfds_mw_workspace_bytes(B.plan));
    }
  // global axis bases again (host), restricted to the layer nodes
  Axis1 X, Y;
  if ((rc = axis_setup(Nx, hx, "x", X)) || (rc = axis_setup(Ny, hy, "y", Y))) return bail(rc);
  P->realx = X.real;
  P->realy = Y.real;
  // layer lists per kind (packed node index within the family axis): primary I -> I/2 - 1,
  // dual I -+ 1 -> (I-2)/2, I/2;  and the node lists used by the kernels
  std::vector<int> lxp, lxd, lyp, lyd, nxl, nyl;  // packed indices; node ids (primary list then dual)
  std::vector<unsigned char> isx(Nx, 0), plx(Nx, 0), ply(Ny, 0);
  for (int a = 0; a < n_ix; ++a) {
    const int I = ix[a];
    lxp.push_back(I / 2 - 1);
    lxd.push_back((I - 2) / 2);
    lxd.push_back(I / 2);
    isx[I - 1] = isx[I] = isx[I + 1] = 1;
    plx[I] = 1;
  }
  for (int b = 0; b < n_iy; ++b) {
    const int J = iy[b];
    lyp.push_back(J / 2 - 1);
    lyd.push_back((J - 2) / 2);
    lyd.push_back(J / 2);
    ply[J] = 1;
  }
  P->Kx[0] = (int)lxp.size(); P->Kx[1] = (int)lxd.size();
  P->Ky[0] = (int)lyp.size(); P->Ky[1] = (int)lyd.size();
  for (int v : lxp) nxl.push_back(2 * v + 2);
  for (int v : lxd) nxl.push_back(2 * v + 1);
  for (int v : lyp) nyl.push_back(2 * v + 2);
  for (int v : lyd) nyl.push_back(2 * v + 1);
  // matrices: full F/I per axis and kind, and their layer sub-matrices
  const int nx = D.nx, ny = D.ny;
  auto sub_cols = [](const std::vector<zc>& F, int rows, int cols, const std::vector<int>& idx) {
    std::vector<zc> o((size_t)rows * idx.size());  // F[:, idx]
    for (int r = 0; r < rows; ++r)
      for (size_t q = 0; q < idx.size(); ++q) o[(size_t)r * idx.size() + q] = F[(size_t)r * cols + idx[q]];
    return o;
  };
  auto sub_rows = [](const std::vector<zc>& I, int cols, const std::vector<int>& idx) {
    std::vector<zc> o((size_t)idx.size() * cols);  // I[idx, :]
    for (size_t q = 0; q < idx.size(); ++q)
      for (int c = 0; c < cols; ++c) o[q * cols + c] = I[(size_t)idx[q] * cols + c];
    return o;
  };
  struct M { std::vector<zc> v; bool real; size_t off; };
  std::vector<M> mats;
  auto add = [&](std::vector<zc> v, bool real) { mats.push_back(M{std::move(v), real, 0}); return (int)mats.size() - 1; };
  const int npx = nx - 1, npy = ny - 1;
  const int mFx[2] = {add(X.Fp, X.real), add(X.Fd, X.real)}, mIx[2] = {add(X.Ip, X.real), add(X.Id, X.real)};
  const int mFy[2] = {add(Y.Fp, Y.real), add(Y.Fd, Y.real)}, mIy[2] = {add(Y.Ip, Y.real), add(Y.Id, Y.real)};
  const int mFxs[2] = {add(sub_cols(X.Fp, npx, npx, lxp), X.real), add(sub_cols(X.Fd, nx, nx, lxd), X.real)};
  const int mIxs[2] = {add(sub_rows(X.Ip, npx, lxp), X.real), add(sub_rows(X.Id, nx, lxd), X.real)};
  const int mFys[2] = {add(sub_cols(Y.Fp, npy, npy, lyp), Y.real), add(sub_cols(Y.Fd, ny, ny, lyd), Y.real)};
  const int mIys[2] = {add(sub_rows(Y.Ip, npy, lyp), Y.real), add(sub_rows(Y.Id, ny, lyd), Y.real)};
  size_t o = 0;
  for (auto& m : mats) {
    m.off = o;
    o += al256(std::max<size_t>(1, m.v.size()) * (m.real ? 8 : 16));
  }
  // compact slot layout: x-part [f][3 nlev][ny][Kx], then y-part [f][3 nlev][Ky][nx]
  int64_t cxo[4], cyo[4], c = 0;
  for (int f = 0; f < 4; ++f) { cxo[f] = c; c += (int64_t)3 * D.nlev[f] * ny * P->Kx[fam_xk(f)]; }
  for (int f = 0; f < 4; ++f) { cyo[f] = c; c += (int64_t)3 * D.nlev[f] * P->Ky[fam_yk(f)] * nx; }
  P->compact = std::max<int64_t>(c, 1);
  P->compact_used = c;
  const size_t oCxo = o; o += al256(sizeof(int64_t) * 4);
  const size_t oCyo = o; o += al256(sizeof(int64_t) * 4);
  const size_t oLx = o; o += al256(sizeof(int) * std::max<size_t>(1, nxl.size()));
  const size_t oLy = o; o += al256(sizeof(int) * std::max<size_t>(1, nyl.size()));
  const size_t oIsx = o; o += al256(Nx);
  const size_t oPlx = o; o += al256(Nx);
  const size_t oPly = o; o += al256(Ny);
  std::vector<char> h(o, 0);
  for (auto& m : mats) {
    if (m.real) {
      double* d = reinterpret_cast<double*>(h.data() + m.off);
      for (size_t q = 0; q < m.v.size(); ++q) d[q] = m.v[q].real();
    } else {
      double2* d = reinterpret_cast<double2*>(h.data() + m.off);
      for (size_t q = 0; q < m.v.size(); ++q) d[q] = make_double2(m.v[q].real(), m.v[q].imag());
    }
  }
  memcpy(h.data() + oCxo, cxo, sizeof cxo);
  memcpy(h.data() + oCyo, cyo, sizeof cyo);
  if (!nxl.empty()) memcpy(h.data() + oLx, nxl.data(), sizeof(int) * nxl.size());
  if (!nyl.empty()) memcpy(h.data() + oLy, nyl.data(), sizeof(int) * nyl.size());
  memcpy(h.data() + oIsx, isx.data(), Nx);
  memcpy(h.data() + oPlx, plx.data(), Nx);
  memcpy(h.data() + oPly, ply.data(), Ny);
  if (cudaMalloc(&P->d_tab, o) != cudaSuccess || cudaMemcpy(P->d_tab, h.data(), o, cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(mwfail(LFDS_ENOMEM, "step-5 tables"));
  P->d_cxo = reinterpret_cast<const int64_t*>(P->d_tab + oCxo);
  P->d_cyo = reinterpret_cast<const int64_t*>(P->d_tab + oCyo);
  P->d_lx = reinterpret_cast<const int*>(P->d_tab + oLx);
  P->d_ly = reinterpret_cast<const int*>(P->d_tab + oLy);
  P->d_isx = reinterpret_cast<const unsigned char*>(P->d_tab + oIsx);
  P->d_plx = reinterpret_cast<const unsigned char*>(P->d_tab + oPlx);
  P->d_ply = reinterpret_cast<const unsigned char*>(P->d_tab + oPly);
  // descriptors: buffers B_F = compact r, B_U = stage-1 compact, B_IF = inverse stage-1 compact,
  // B_RED = compact w, B_MS = coefficients (x-part), B_T1 = coefficients (y-part)
  auto ao = [&](int m) { return (int64_t)(mats[m].off / (mats[m].real ? 8 : 16)); };
  std::vector<lfds::GemmDesc> desc;
  const int64_t pl = D.plane;
  for (int g = 0; g < 8; ++g) {
    for (int f = 0; f < 4; ++f) {
      const int xk = fam_xk(f), yk = fam_yk(f);
      const int nxf = xk ? nx : nx - 1, nyf = yk ? ny : ny - 1;
      const int Kx = P->Kx[xk], Ky = P->Ky[yk];
      const int64_t nl = 3 * D.nlev[f];
      lfds::GemmDesc d{};
      d.N1 = (int)nl;
      switch (g) {
        case 0:  // XA: Y1[m][kx] = Fy RXc
          d.a_off = ao(mFy[yk]); d.sAi = nyf; d.sAj = 1; d.M = d.K = nyf;
          d.b_buf = lfds::B_F; d.b_off = cxo[f]; d.sBj = Kx; d.sB1 = (int64_t)ny * Kx; d.sB2 = 1; d.N2 = Kx;
          d.c_buf = lfds::B_U; d.c_off = cxo[f] + (yk ? 0 : Kx); d.sCi = Kx; d.sC1 = (int64_t)ny * Kx; d.sC2 = 1;
          break;
        case 1:  // XB: coef[m][l] = sum_kx Y1[m][kx] Fx[l, layer kx]
          d.a_off = ao(mFxs[xk]); d.sAi = Kx; d.sAj = 1; d.M = nxf; d.K = Kx;
          d.b_buf = lfds::B_U; d.b_off = cxo[f]; d.sBj = 1; d.sB1 = (int64_t)ny * Kx; d.sB2 = Kx; d.N2 = ny;
          d.c_buf = lfds::B_MS; d.c_off = D.fam_off[f] + (xk ? 0 : 1); d.sCi = 1; d.sC1 = pl; d.sC2 = nx;
          break;
        case 2:  // YA: X1[ky][l] = RYc Fx^T
          d.a_off = ao(mFx[xk]); d.sAi = nxf; d.sAj = 1; d.M = d.K = nxf;
          d.b_buf = lfds::B_F; d.b_off = cyo[f]; d.sBj = 1; d.sB1 = (int64_t)Ky * nx; d.sB2 = nx; d.N2 = Ky;
          d.c_buf = lfds::B_U; d.c_off = cyo[f] + (xk ? 0 : 1); d.sCi = 1; d.sC1 = (int64_t)Ky * nx; d.sC2 = nx;
          break;
        case 3:  // YB: coef2[m][l] = sum_ky Fy[m, layer ky] X1[ky][l]
          d.a_off = ao(mFys[yk]); d.sAi = Ky; d.sAj = 1; d.M = nyf; d.K = Ky;
          d.b_buf = lfds::B_U; d.b_off = cyo[f]; d.sBj = nx; d.sB1 = (int64_t)Ky * nx; d.sB2 = 1; d.N2 = nx;
          d.c_buf = lfds::B_T1; d.c_off = D.fam_off[f] + (yk ? 0 : nx); d.sCi = nx; d.sC1 = pl; d.sC2 = 1;
          break;
        case 4:  // IXA: Z1[m][kx] = sum_l Ix[layer kx, l] w~[m][l]
          d.a_off = ao(mIxs[xk]); d.sAi = nxf; d.sAj = 1; d.M = Kx; d.K = nxf;
          d.b_buf = lfds::B_MS; d.b_off = D.fam_off[f] + (xk ? 0 : 1); d.sBj = 1; d.sB1 = pl; d.sB2 = nx; d.N2 = ny;
          d.c_buf = lfds::B_IF; d.c_off = cxo[f]; d.sCi = 1; d.sC1 = (int64_t)ny * Kx; d.sC2 = Kx;
          break;
        case 5:  // IXB: WXc[y][kx] = Iy Z1
          d.a_off = ao(mIy[yk]); d.sAi = nyf; d.sAj = 1; d.M = d.K = nyf;
          d.b_buf = lfds::B_IF; d.b_off = cxo[f] + (yk ? 0 : Kx); d.sBj = Kx; d.sB1 = (int64_t)ny * Kx; d.sB2 = 1;
          d.N2 = Kx;
          d.c_buf = lfds::B_RED; d.c_off = cxo[f]; d.sCi = Kx; d.sC1 = (int64_t)ny * Kx; d.sC2 = 1;
          break;
        case 6:  // IYA: Z2[ky][l] = sum_m Iy[layer ky, m] w~[m][l]
          d.a_off = ao(mIys[yk]); d.sAi = nyf; d.sAj = 1; d.M = Ky; d.K = nyf;
          d.b_buf = lfds::B_MS; d.b_off = D.fam_off[f] + (yk ? 0 : nx); d.sBj = nx; d.sB1 = pl; d.sB2 = 1; d.N2 = nx;
          d.c_buf = lfds::B_IF; d.c_off = cyo[f]; d.sCi = nx; d.sC1 = (int64_t)Ky * nx; d.sC2 = 1;
          break;
        default:  // IYB: WYc[ky][x] = Z2 Ix^T
          d.a_off = ao(mIx[xk]); d.sAi = nxf; d.sAj = 1; d.M = d.K = nxf;
          d.b_buf = lfds::B_IF; d.b_off = cyo[f] + (xk ? 0 : 1); d.sBj = 1; d.sB1 = (int64_t)Ky * nx; d.sB2 = nx;
          d.N2 = Ky;
          d.c_buf = lfds::B_RED; d.c_off = cyo[f]; d.sCi = 1; d.sC1 = (int64_t)Ky * nx; d.sC2 = nx;
          break;
      }
      desc.push_back(d);
      P->gM[g] = std::max(P->gM[g], d.M);
      P->gN[g] = std::max<int64_t>(P->gN[g], (int64_t)d.N1 * d.N2);
    }
    const bool xaxis = g == 1 || g == 2 || g == 4 || g == 7;  // contractions along x use x's bases
    P->gReal[g] = xaxis ? X.real : Y.real;
    P->gKc[g] = (g == 1 || g == 2 || g == 4 || g == 7);     // K index contiguous in B
  }
  if (cudaMalloc(&P->d_desc, desc.size() * sizeof(lfds::GemmDesc)) != cudaSuccess ||
      cudaMemcpy(P->d_desc, desc.data(), desc.size() * sizeof(lfds::GemmDesc), cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(mwfail(LFDS_ECUDA, "descriptor upload"));
  *out = P.release();
  return LFDS_OK;
}

static size_t mw2_layout(const lfds_mw2* P, size_t off[8]) {
  const MwDev& D = P->glob->D;
  const size_t full = al256((size_t)3 * D.Nz * D.Ny * D.Nx * 16);
  const size_t fam = al256(P->glob->fam_elems * 16), cp = al256(P->glob->cp_elems * 16);
  const size_t cmp = al256((size_t)P->compact * 16), sub = al256(P->sub_elems * 16);
  size_t o = 0;
  off[0] = o; o += full;          // r, then f2
  off[1] = o; o += full;          // E
  off[2] = o; o += 2 * fam + cp;  // coef, coef2, Thomas scratch
  off[3] = o; o += 4 * cmp;       // compact slots
  off[4] = o; o += sub;           // block f
  off[5] = o; o += sub;           // block H
  off[6] = o; o += al256(P->sub_ws);
  return o;
}

size_t lfds_mw2_workspace_bytes(const lfds_mw2* P) {
  if (!P) return 0;
  size_t off[8];
  return mw2_layout(P, off);
}

static cudaError_t box_copy(const lfds_mw2::Blk& B, const MwDev& D, void* full, void* packed, bool to_packed,
                            bool interior, cudaStream_t st) {
  const int bx = B.x1 - B.x0 + 1, by = B.y1 - B.y0 + 1;
  const int e = interior ? 1 : 0;
  cudaMemcpy3DParms p{};
  p.extent = make_cudaExtent((size_t)(bx - 2 * e) * 16, by - 2 * e, (size_t)3 * D.Nz);
  p.kind = cudaMemcpyDeviceToDevice;
  cudaPitchedPtr F = make_cudaPitchedPtr(full, (size_t)D.Nx * 16, (size_t)D.Nx * 16, D.Ny);
  cudaPitchedPtr S = make_cudaPitchedPtr(packed, (size_t)bx * 16, (size_t)bx * 16, by);
  const cudaPos pf = make_cudaPos((size_t)(B.x0 + e) * 16, B.y0 + e, 0), ps = make_cudaPos((size_t)e * 16, e, 0);
  if (to_packed) { p.srcPtr = F; p.srcPos = pf; p.dstPtr = S; p.dstPos = ps; }
  else { p.srcPtr = S; p.srcPos = ps; p.dstPtr = F; p.dstPos = pf; }
  return cudaMemcpy3DAsync(&p, st);
}

int lfds_mw2_solve(lfds_mw2* P, const void* f_dev, void* h_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!P || !f_dev || !h_dev || !ws) return mwfail(LFDS_EINVAL, "bad arguments");
  size_t off[8];
  if (ws_bytes < mw2_layout(P, off)) return mwfail(LFDS_EINVAL, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  (void)cudaGetLastError();
  const MwDev& D = P->glob->D;
  char* w = static_cast<char*>(ws);
  double2* R = reinterpret_cast<double2*>(w + off[0]);
  double2* E = reinterpret_cast<double2*>(w + off[1]);
  double2* coef = reinterpret_cast<double2*>(w + off[2]);
  double2* coef2 = coef + al256(P->glob->fam_elems * 16) / 16;
  double2* cp = coef2 + al256(P->glob->fam_elems * 16) / 16;
  const size_t cmp = al256((size_t)P->compact * 16);
  char* sf = w + off[4];
  char* sh = w + off[5];
  void* sws = w + off[6];
  double2* H = static_cast<double2*>(h_dev);
  const double2* F = static_cast<const double2*>(f_dev);
  const int64_t N = (int64_t)D.Nz * D.Ny * D.Nx;
  const unsigned gs = (unsigned)std::min<int64_t>((N + 255) / 256, 148 * 16);
  int rc;
  auto cuda = [&](cudaError_t x) { return x == cudaSuccess ? LFDS_OK : mwfail(LFDS_ECUDA, "two-level: %s", cudaGetErrorString(x)); };
  auto blocks = [&](const void* src) -> int {
    for (auto& B : P->blk) {
      int q;
      if ((q = cuda(box_copy(B, D, const_cast<void*>(src), sf, true, false, st)))) return q;
      if ((q = lfds_mw_solve(B.plan, sf, sh, sws, P->sub_ws, stream))) return q;
      if ((q = cuda(box_copy(B, D, H, sh, false, true, st)))) return q;
    }
    return LFDS_OK;
  };
  // 1-3: v on every block, zero on the planes
  if ((rc = cuda(cudaMemsetAsync(H, 0, (size_t)3 * N * 16, st)))) return rc;
  if ((rc = blocks(F))) return rc;
  // 4: r = f - A_h v
  k_mw_curlh<<<gs, 256, 0, st>>>(D, H, E);
  k_mw_curle<<<gs, 256, 0, st>>>(D, E, H, F, R);
  // 5: w on the layers
  lfds::Bufs b{};
  b.p[lfds::B_TAB] = P->d_tab;
  b.p[lfds::B_F] = w + off[3];
  b.p[lfds::B_U] = w + off[3] + cmp;
  b.p[lfds::B_IF] = w + off[3] + 2 * cmp;
  b.p[lfds::B_RED] = w + off[3] + 3 * cmp;
  b.p[lfds::B_MS] = coef;
  b.p[lfds::B_T1] = coef2;
  const int64_t ctot = P->compact_used;
  const unsigned gc = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ctot + 255) / 256, 148 * 16));
  if (ctot) k_mw2_gather_r<<<gc, 256, 0, st>>>(D, R, static_cast<double2*>(b.p[lfds::B_F]), P->d_cxo, P->d_cyo, P->d_lx,
                                     P->d_ly, P->Kx[0], P->Kx[1], P->Ky[0], P->Ky[1], P->d_isx, ctot);
  if ((rc = cuda(cudaGetLastError()))) return rc;
  auto group = [&](int g) {  // (empty when the axis has no interfaces; XB / YB then write zeros)
    if (P->gM[g] == 0 || P->gN[g] == 0) return cudaSuccess;
    return lfds::launch_xform(P->d_desc + 4 * g, 4, P->gM[g], P->gN[g], P->gReal[g], P->gKc[g], b, st);
  };
  for (int g = 0; g < 4; ++g)
    if ((rc = cuda(group(g)))) return rc;
  mw_zsolve_launch(D, coef, cp, coef2, st);
  if ((rc = cuda(cudaGetLastError()))) return rc;
  for (int g = 4; g < 8; ++g)
    if ((rc = cuda(group(g)))) return rc;
  if (ctot) k_mw2_add_w<<<gc, 256, 0, st>>>(D, static_cast<const double2*>(b.p[lfds::B_RED]), H, P->d_cxo, P->d_cyo, P->d_lx,
                                  P->d_ly, P->Kx[0], P->Kx[1], P->Ky[0], P->Ky[1], P->d_isx, ctot);
  // 6: interface data lifted into the right side (into R)
  k_mw2_elift<<<gs, 256, 0, st>>>(D, H, E, P->d_plx, P->d_ply);
  k_mw2_flift<<<gs, 256, 0, st>>>(D, E, F, R, P->d_plx, P->d_ply);
  if ((rc = cuda(cudaGetLastError()))) return rc;
  // 7: every block with its interface data; H = w stays on the plane P nodes
  if ((rc = blocks(R))) return rc;
  return cuda(cudaGetLastError());
}

int lfds_mw2_blocks(const lfds_mw2* P, int* n) {
  if (!P || !n) return mwfail(LFDS_EINVAL, "bad arguments");
  *n = (int)P->blk.size();
  return LFDS_OK;
}

}  // extern "C"
