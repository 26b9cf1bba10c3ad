// Batched z tridiagonal solves of the blocked separable method (arXiv 1909.01299):
//   step 2  T_lm v~_lm = f~_lm in every block, in place      (k_zs1)
//   step 6    T_lm w~_lm = l~_lm (Dirichlet lifting, reading R8),
//                              solution added to v~ in place                      (k_zs2)
//   step 5    T_lm w^_lm = r^_lm for every global mode, with the
//                              rank-|I| right side r^ built on the fly            (k_zs3)
// with T_lm = A_z + lambda M_z + (lambda_l + mu_m) M_z^sigma (reading R1).
//
// One thread per z-line; a CTA covers a TL x TM tile of (l, m) modes (l fastest), so a
// warp's row access is TL consecutive complex numbers (one 512-B segment for TL = 32).
// Mode space is [r][k][m][l]: a z-line is strided by nx*ny.
//
// Thomas elimination without pivoting (reading R15):
//   forward   r_k = b_k - a_k c'_{k-1},  c'_k = c_k / r_k,  d'_k = (d_k - a_k d'_{k-1}) / r_k
//   backward  x_k = d'_k - c'_k x_{k+1}
// c' and d' never go to memory in full: the forward sweep stores a (c', d') checkpoint at
// the start of every ZSEG-row segment (global scratch, L2-resident while the CTA lives);
// the backward sweep recomputes a segment from its checkpoint into registers.
//   k_zs1 re-reads the RHS in the backward sweep (48 B/unknown of HBM traffic);
//   k_zs2 rebuilds its RHS from the four face transforms and reads/writes v~ once
//         (32 B/unknown);
//   k_zs3 builds its RHS once, stores d' in the global mode array (the only copy of the
//         line) and only recomputes c' backwards (48 B/unknown, no separate RHS pass).
// Rows of a thread's own line come through per-thread cp.async copies into a private
// shared-memory ring, NSTAGE-1 segments ahead.  Rows shared by the CTA (face transforms,
// interface residual rows) are staged cooperatively, double-buffered, one segment ahead,
// so no load sits inside a dependency chain.  k_zs3 forms its right-hand side tile
//   r^[k][m][l] = sum_a R1[a][k][m] W_x[I_a][l] + sum_b W_y[I_b][m] R2[b][k][l]
// (a rank-|I| complex contraction) on the DMMA tensor pipe from the staged rows.
// A pivot monitor keeps min |r_k|^2 / (|b_k|^2 + (|a_k|+|c_k|)^2) (reported as its sqrt).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "lfds_internal.h"

namespace lfds {
namespace {

struct cplx {
  double x, y;
};
__device__ __forceinline__ cplx mk(double a, double b) { return cplx{a, b}; }
__device__ __forceinline__ cplx mk(double2 v) { return cplx{v.x, v.y}; }
__device__ __forceinline__ cplx ld(const double2* p) {
  const double2 v = __ldg(p);
  return cplx{v.x, v.y};
}
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return cplx{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return cplx{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
  return cplx{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {  // a*b + c
  return cplx{fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
__device__ __forceinline__ double cabs1(cplx a) { return fabs(a.x) + fabs(a.y); }
// reciprocal from the MUFU.RCP64H seed and two Newton steps (full fp64 accuracy)
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ void atomic_min_pos(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int ZT = 256;  // threads per CTA

// staged z tables (real tables: ag[k] = (a, g), ce[k] = (c, e), m2[k] = (|a|+|c|)^2;
// complex tables: sa, sg, sc, se)
struct ZTabS {
  const double2 *ag, *ce, *sa, *sg, *sc, *se;
  const double* m2;
};

// Row types: RT 0 = complex z table; RT 1 = real z table, complex shift s = lambda_l + mu_m;
// RT 2 = real z table and real shift (both block bases real: U or R blocks), where c' is real
// and the elimination costs about half.
template <int RT>
__device__ __forceinline__ void zrow(const ZTabS& T, int k, cplx s, cplx& a, cplx& b, cplx& c, double& m2) {
  if (RT >= 1) {
    const double2 ag = T.ag[k], ce = T.ce[k];
    a = mk(ag.x, 0);
    c = mk(ce.x, 0);
    b = mk(fma(s.x, ce.y, ag.y), RT == 2 ? 0.0 : s.y * ce.y);
    m2 = T.m2[k];
  } else {
    const double2 a2 = T.sa[k], g2 = T.sg[k], c2 = T.sc[k], e2 = T.se[k];
    a = mk(a2.x, a2.y);
    c = mk(c2.x, c2.y);
    b = cfma(s, mk(e2.x, e2.y), mk(g2.x, g2.y));
    const double t = cabs1(a) + cabs1(c);
    m2 = t * t;
  }
}

// one forward elimination row; returns |r|^2
template <int RT>
__device__ __forceinline__ double elim(cplx a, cplx b, cplx c, cplx d, cplx& cp, cplx& dp) {
  if (RT == 2) {
    const double r = fma(-a.x, cp.x, b.x);
    const double in = fast_rcp(r);
    cp = mk(c.x * in, 0);
    dp = mk(fma(-a.x, dp.x, d.x) * in, fma(-a.x, dp.y, d.y) * in);
    return r * r;
  }
  cplx r, t;
  if (RT == 1) {
    r = mk(fma(-a.x, cp.x, b.x), fma(-a.x, cp.y, b.y));
    t = mk(fma(-a.x, dp.x, d.x), fma(-a.x, dp.y, d.y));
  } else {
    r = b - a * cp;
    t = d - a * dp;
  }
  const double n2 = fma(r.x, r.x, r.y * r.y);
  const double in = fast_rcp(n2);
  const cplx inv = mk(r.x * in, -r.y * in);
  cp = RT == 1 ? mk(c.x * inv.x, c.x * inv.y) : c * inv;
  dp = t * inv;
  return n2;
}
// c' only (k_zs3 backward recompute)
template <int RT>
__device__ __forceinline__ void elim_c(cplx a, cplx b, cplx c, cplx& cp) {
  if (RT == 2) {
    cp = mk(c.x * fast_rcp(fma(-a.x, cp.x, b.x)), 0);
    return;
  }
  cplx r;
  if (RT == 1) r = mk(fma(-a.x, cp.x, b.x), fma(-a.x, cp.y, b.y));
  else r = b - a * cp;
  const double in = fast_rcp(fma(r.x, r.x, r.y * r.y));
  const cplx inv = mk(r.x * in, -r.y * in);
  cp = RT == 1 ? mk(c.x * inv.x, c.x * inv.y) : c * inv;
}
// back substitution x_k = d'_k - c'_k x_{k+1}
template <int RT>
__device__ __forceinline__ cplx backsub(cplx d, cplx c, cplx x) {
  if (RT == 2) return mk(fma(-c.x, x.x, d.x), fma(-c.x, x.y, d.y));
  return d - c * x;
}

__host__ __device__ __forceinline__ int ztab_slots(int nz, bool realz) {  // in double2 units
  return realz ? 2 * nz + (nz + 1) / 2 : 4 * nz;
}

template <bool REALZ>
__device__ __forceinline__ ZTabS stage_ztab(ZTab tab, const double2* TAB, int nz, double2* zsm) {
  ZTabS T{};
  if (REALZ) {
    double2* ag = zsm;
    double2* ce = zsm + nz;
    double* m2 = reinterpret_cast<double*>(zsm + 2 * nz);
    for (int k = threadIdx.x; k < nz; k += blockDim.x) {
      const double a = TAB[tab.a + k].x, c = TAB[tab.c + k].x;
      ag[k] = make_double2(a, TAB[tab.g + k].x);
      ce[k] = make_double2(c, TAB[tab.e + k].x);
      m2[k] = (fabs(a) + fabs(c)) * (fabs(a) + fabs(c));
    }
    T.ag = ag; T.ce = ce; T.m2 = m2;
  } else {
    double2* s = zsm;
    for (int k = threadIdx.x; k < nz; k += blockDim.x) {
      s[k] = TAB[tab.a + k];
      s[nz + k] = TAB[tab.g + k];
      s[2 * nz + k] = TAB[tab.c + k];
      s[3 * nz + k] = TAB[tab.e + k];
    }
    T.sa = s; T.sg = s + nz; T.sc = s + 2 * nz; T.se = s + 3 * nz;
  }
  return T;
}

// per-thread ring of ZSEG-row segments of one z-line
template <int ZSEG, int NSTAGE, bool FULL = false>
struct Ring {
  double2* s;  // s[(slot * ZSEG + j) * ZT + tid]
  const double2* line;
  int64_t stride;
  int nz;
  bool active;
  __device__ __forceinline__ void issue(int seg) const {
    if (active && seg >= 0) {
      double2* d = s + (seg % NSTAGE) * ZSEG * ZT + threadIdx.x;
      const int k0 = seg * ZSEG;
#pragma unroll
      for (int j = 0; j < ZSEG; ++j)
        if (FULL || k0 + j < nz) cp16(d + j * ZT, line + (int64_t)(k0 + j) * stride);
    }
    cp_commit();
  }
  __device__ __forceinline__ cplx get(int seg, int j) const {
    return mk(s[((seg % NSTAGE) * ZSEG + j) * ZT + threadIdx.x]);
  }
};

struct Tile {  // the CTA's (l, m) tile and this thread's line
  int l0, m0, l, m;
  bool active;
};
template <int TL>
__device__ __forceinline__ bool make_tile(const ZBlock& B, Tile& t) {
  constexpr int TM = ZT / TL;
  const int tiles_l = (B.nx + TL - 1) / TL;
  const int tl = blockIdx.x % tiles_l, tm = blockIdx.x / tiles_l;
  t.l0 = tl * TL;
  t.m0 = tm * TM;
  if (t.m0 >= B.ny) return false;
  t.l = t.l0 + (int)(threadIdx.x % TL);
  t.m = t.m0 + (int)(threadIdx.x / TL);
  t.active = t.l < B.nx && t.m < B.ny;
  return true;
}

__device__ __forceinline__ void commit_minpiv(float v, double* out) {
  if (!out) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomic_min_pos(out, (double)sqrtf(v));
}

__device__ __forceinline__ double2* ck_base(const Bufs& bufs) {
  return reinterpret_cast<double2*>(bufs.p[B_CK]) +
         (((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * ZT + threadIdx.x;
}

// ===================================================================== step 2
template <int RT, bool FULL, int TL>
__device__ __forceinline__ void zs1_body(const ZBlock& B, const Tile& t, int nz, const ZTabS& T,
                                         const double2* TAB, Bufs& bufs, double2* ring_smem, double* minpiv_out) {
  constexpr int ZSEG = 8, NSTAGE = 3;
  const int r = blockIdx.z;
  const int64_t nxy = (int64_t)B.nx * B.ny;
  double2* line = reinterpret_cast<double2*>(bufs.p[B.buf]) + B.ms_off + (int64_t)r * nz * nxy +
                  (int64_t)(t.active ? t.m : 0) * B.nx + (t.active ? t.l : 0);
  const Ring<ZSEG, NSTAGE, FULL> ring{ring_smem, line, nxy, nz, t.active};
  const int nseg = (nz + ZSEG - 1) / ZSEG;
  const int64_t nslot = (int64_t)gridDim.x * gridDim.y * gridDim.z * ZT;
  double2* ck = ck_base(bufs);
  float minpiv = 1.0f;
  const cplx s = t.active ? ld(TAB + B.lamx + t.l) + ld(TAB + B.lamy + t.m) : mk(0, 0);
  cplx cp = mk(0, 0), dp = mk(0, 0);
#pragma unroll
  for (int q = 0; q < NSTAGE - 1; ++q) ring.issue(q < nseg ? q : -1);
  for (int sg = 0; sg < nseg; ++sg) {
    const int k0 = sg * ZSEG;
    ring.issue(sg + NSTAGE - 1 < nseg ? sg + NSTAGE - 1 : -1);
    cp_wait<NSTAGE - 1>();
    if (!t.active) continue;
    ck[(int64_t)(2 * sg) * nslot] = make_double2(cp.x, cp.y);
    ck[(int64_t)(2 * sg + 1) * nslot] = make_double2(dp.x, dp.y);
#pragma unroll
    for (int j = 0; j < ZSEG; ++j) {
      const int k = k0 + j;
      if (FULL || k < nz) {
        cplx a, b, c;
        double m2;
        zrow<RT>(T, k, s, a, b, c, m2);
        const double n2 = elim<RT>(a, b, c, ring.get(sg, j), cp, dp);
        minpiv = fminf(minpiv, __fdividef((float)n2, (float)fma(b.x, b.x, fma(b.y, b.y, m2))));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NSTAGE - 1; ++q) ring.issue(nseg - 1 - q);
  cplx x = mk(0, 0);
  double2 nc = ck[(int64_t)(2 * (nseg - 1)) * nslot], nd = ck[(int64_t)(2 * (nseg - 1) + 1) * nslot];
  for (int sg = nseg - 1; sg >= 0; --sg) {
    const int k0 = sg * ZSEG;
    ring.issue(sg - (NSTAGE - 1));
    cp_wait<NSTAGE - 1>();
    if (!t.active) continue;
    cplx rb[ZSEG], cs[ZSEG];
    cplx cc = mk(nc), dd = mk(nd);
    if (sg > 0) {  // next segment's checkpoint in flight while this one is solved
      nc = ck[(int64_t)(2 * sg - 2) * nslot];
      nd = ck[(int64_t)(2 * sg - 1) * nslot];
    }
#pragma unroll
    for (int j = 0; j < ZSEG; ++j) {
      const int k = k0 + j;
      rb[j] = mk(0, 0);
      if (FULL || k < nz) {
        cplx a, b, c;
        double m2;
        zrow<RT>(T, k, s, a, b, c, m2);
        elim<RT>(a, b, c, ring.get(sg, j), cc, dd);
        rb[j] = dd;
      }
      cs[j] = cc;
    }
    double2* lp = line + (int64_t)k0 * nxy;
#pragma unroll
    for (int j = ZSEG - 1; j >= 0; --j) {
      if (FULL || k0 + j < nz) {
        x = backsub<RT>(rb[j], cs[j], x);
        lp[j * nxy] = make_double2(x.x, x.y);
      }
    }
  }
  cp_wait<0>();
  commit_minpiv(minpiv, minpiv_out);
}

template <bool REALZ, int TL, bool FULL>
__global__ void __launch_bounds__(ZT, 2) k_zs1(const ZBlock* __restrict__ blocks, int nz, ZTab tab, Bufs bufs,
                                               double* minpiv_out) {
  extern __shared__ __align__(16) double2 zsm[];
  const ZBlock B = blocks[blockIdx.y];
  Tile t;
  if (!make_tile<TL>(B, t)) return;  // whole CTA, before any barrier
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const ZTabS T = stage_ztab<REALZ>(tab, TAB, nz, zsm);
  __syncthreads();
  double2* ring = zsm + ztab_slots(nz, REALZ);
  if (!REALZ) zs1_body<0, FULL, TL>(B, t, nz, T, TAB, bufs, ring, minpiv_out);
  else if (B.pad_) zs1_body<2, FULL, TL>(B, t, nz, T, TAB, bufs, ring, minpiv_out);  // real shift
  else zs1_body<1, FULL, TL>(B, t, nz, T, TAB, bufs, ring, minpiv_out);
}

// ===================================================================== step 6
// Face rows staged per segment, separate arrays per face: GL[j][TM], GR[j][TM] (indexed
// by m), GB[j][TL], GT[j][TL] (indexed by l).  Every thread owns fixed copy slots (shift/mask
// index math only): 2*ZSEG*(TL+TM) copies over ZT threads.  The -sigma_k factor of the lifting
// is folded into the rows of the z table the step-6 solve uses (row scaling leaves the
// solution and the c'/d' recurrences unchanged).
template <int TL, int ZSEG>
struct FaceStage {
  static constexpr int TM = ZT / TL;
  static constexpr int GB = 0, GT = ZSEG * TL, GL = 2 * ZSEG * TL, GR = GL + ZSEG * TM;
  static constexpr int SLOTS = GR + ZSEG * TM;  // double2 per stage
};

template <int RT, bool FULL, int TL>
__device__ __forceinline__ void zs2_body(const ZBlock& B, const Tile& t, int nz, const ZTabS& T, const double2* TAB,
                                         Bufs& bufs, double2* fsm) {
  // 8-row solve segments; the face rows are staged 16 rows (two segments) at a time, so the
  // CTA meets at a barrier twice per 16 rows instead of twice per 8
  constexpr int ZSEG = 8, FSEG = 2 * ZSEG, NSTAGE = 2, TM = ZT / TL;
  using FS = FaceStage<TL, FSEG>;
  const int r = blockIdx.z;
  const double2* IF = reinterpret_cast<const double2*>(bufs.p[B_IF]);
  const int64_t nxy = (int64_t)B.nx * B.ny;
  double2* line = reinterpret_cast<double2*>(bufs.p[B_MS]) + B.ms_off + (int64_t)r * nz * nxy +
                  (int64_t)(t.active ? t.m : 0) * B.nx + (t.active ? t.l : 0);
  const Ring<ZSEG, NSTAGE, FULL> ring{fsm + 2 * FS::SLOTS, line, nxy, nz, t.active};
  const int nseg = (nz + ZSEG - 1) / ZSEG, nfs = (nz + FSEG - 1) / FSEG;
  const int64_t nslot = (int64_t)gridDim.x * gridDim.y * gridDim.z * ZT;
  double2* ck = ck_base(bufs);
  // face f row k at IF[base_f + (r*nz + k)*fs + index]
  const int64_t fs = B.fstride, ro = (int64_t)r * nz * fs;
  const bool hL = B.gL >= 0, hR = B.gR >= 0, hB = B.gB >= 0, hT = B.gT >= 0;
  // cooperative copy of face segment q (rows 16q .. 16q+15) into slot q&1
  auto stage = [&](int q) {
    if (q >= 0 && q < nfs) {
      double2* d = fsm + (q & 1) * FS::SLOTS;
      const int k0 = q * FSEG;
#pragma unroll
      for (int i = 0; i < (FS::SLOTS + ZT - 1) / ZT; ++i) {
        const int c = threadIdx.x + i * ZT;
        if (c >= FS::SLOTS) break;
        const double2* src = nullptr;
        if (c < FS::GL) {  // GB / GT rows, TL entries each
          const int f = c / (FSEG * TL), j = (c / TL) % FSEG, li = c % TL, k = k0 + j;
          if (k < nz && t.l0 + li < B.nx && (f ? hT : hB)) src = IF + (f ? B.gT : B.gB) + ro + k * fs + t.l0 + li;
        } else {  // GL / GR rows, TM entries each
          const int c2 = c - FS::GL;
          const int f = c2 / (FSEG * TM), j = (c2 / TM) % FSEG, mi = c2 % TM, k = k0 + j;
          if (k < nz && t.m0 + mi < B.ny && (f ? hR : hL)) src = IF + (f ? B.gR : B.gL) + ro + k * fs + t.m0 + mi;
        }
        if (src) cp16(d + c, src);
      }
    }
    cp_commit();
  };
  const cplx cL = hL && t.active ? mk(B.cL) * ld(TAB + B.wx0 + t.l) : mk(0, 0);
  const cplx cR = hR && t.active ? mk(B.cR) * ld(TAB + B.wx1 + t.l) : mk(0, 0);
  const cplx cB = hB && t.active ? mk(B.cB) * ld(TAB + B.wy0 + t.m) : mk(0, 0);
  const cplx cT = hT && t.active ? mk(B.cT) * ld(TAB + B.wy1 + t.m) : mk(0, 0);
  const int tx = threadIdx.x % TL, ty = threadIdx.x / TL;
  // l~(k) = -sigma_k (cL_l GL[k][m] + cR_l GR[k][m] + cB_m GB[k][l] + cT_m GT[k][l]); the
  // -sigma_k is in the (row-scaled) z table, so the right side is the bracket.  Real-basis
  // blocks (RT 2: real steps, so real W rows and real face couplings) take real coefficients:
  // 2 FMAs per face term instead of 4.
  auto lift = [&](int sg, int j) {
    const double2* d = fsm + ((sg >> 1) & 1) * FS::SLOTS;
    const int jj = (sg & 1) * ZSEG + j;
    cplx acc = mk(0, 0);
    if (RT == 2) {
      auto rfma = [](double c, double2 v, cplx a) { return mk(fma(c, v.x, a.x), fma(c, v.y, a.y)); };
      if (hL) acc = rfma(cL.x, d[FS::GL + jj * TM + ty], acc);
      if (hR) acc = rfma(cR.x, d[FS::GR + jj * TM + ty], acc);
      if (hB) acc = rfma(cB.x, d[FS::GB + jj * TL + tx], acc);
      if (hT) acc = rfma(cT.x, d[FS::GT + jj * TL + tx], acc);
      return acc;
    }
    if (hL) acc = cfma(cL, mk(d[FS::GL + jj * TM + ty]), acc);
    if (hR) acc = cfma(cR, mk(d[FS::GR + jj * TM + ty]), acc);
    if (hB) acc = cfma(cB, mk(d[FS::GB + jj * TL + tx]), acc);
    if (hT) acc = cfma(cT, mk(d[FS::GT + jj * TL + tx]), acc);
    return acc;
  };
  const cplx s = t.active ? ld(TAB + B.lamx + t.l) + ld(TAB + B.lamy + t.m) : mk(0, 0);
  // ---- forward sweep
  cplx cp = mk(0, 0), dp = mk(0, 0);
  stage(0);
  for (int sg = 0; sg < nseg; ++sg) {
    const int k0 = sg * ZSEG;
    if ((sg & 1) == 0) {  // first segment of face segment sg/2
      stage((sg >> 1) + 1);
      cp_wait<1>();
      __syncthreads();  // face segment staged by every thread
    }
    if (t.active) {
      ck[(int64_t)(2 * sg) * nslot] = make_double2(cp.x, cp.y);
      ck[(int64_t)(2 * sg + 1) * nslot] = make_double2(dp.x, dp.y);
#pragma unroll
      for (int j = 0; j < ZSEG; ++j) {
        const int k = k0 + j;
        if (FULL || k < nz) {
          cplx a, b, c;
          double m2;
          zrow<RT>(T, k, s, a, b, c, m2);
          elim<RT>(a, b, c, lift(sg, j), cp, dp);  // same T_lm as step 2: pivots monitored there
        }
      }
    }
    if ((sg & 1) == 1 || sg == nseg - 1) __syncthreads();  // slot consumed before it is refilled
  }
  // ---- backward sweep: faces staged again in reverse order, v~ through the ring
  cp_wait<0>();
  stage((nseg - 1) >> 1);
  ring.issue(nseg - 1);
  cplx x = mk(0, 0);
  double2 nc = ck[(int64_t)(2 * (nseg - 1)) * nslot], nd = ck[(int64_t)(2 * (nseg - 1) + 1) * nslot];
  for (int sg = nseg - 1; sg >= 0; --sg) {
    const int k0 = sg * ZSEG;
    const bool first = (sg & 1) == 1 || sg == nseg - 1;  // first visited segment of its face segment
    if (first) stage((sg >> 1) - 1);
    else cp_commit();
    ring.issue(sg - 1);
    cp_wait<2>();  // this face segment and this segment's ring rows, issued earlier
    if (first) __syncthreads();
    if (t.active) {
      cplx rb[ZSEG], cs[ZSEG];
      cplx cc = mk(nc), dd = mk(nd);
      if (sg > 0) {
        nc = ck[(int64_t)(2 * sg - 2) * nslot];
        nd = ck[(int64_t)(2 * sg - 1) * nslot];
      }
#pragma unroll
      for (int j = 0; j < ZSEG; ++j) {
        const int k = k0 + j;
        rb[j] = mk(0, 0);
        if (FULL || k < nz) {
          cplx a, b, c;
          double m2;
          zrow<RT>(T, k, s, a, b, c, m2);
          elim<RT>(a, b, c, lift(sg, j), cc, dd);
          rb[j] = dd;
        }
        cs[j] = cc;
      }
      double2* lp = line + (int64_t)k0 * nxy;
#pragma unroll
      for (int j = ZSEG - 1; j >= 0; --j) {
        if (FULL || k0 + j < nz) {
          x = backsub<RT>(rb[j], cs[j], x);
          const cplx o = ring.get(sg, j);
          lp[j * nxy] = make_double2(o.x + x.x, o.y + x.y);
        }
      }
    }
    if ((sg & 1) == 0) __syncthreads();  // face slot consumed before it is refilled
  }
  cp_wait<0>();
}


template <bool REALZ, int TL, bool FULL>
__global__ void __launch_bounds__(ZT, 2) k_zs2(const ZBlock* __restrict__ blocks, int nz, ZTab tab, Bufs bufs) {
  extern __shared__ __align__(16) double2 zsm[];
  const ZBlock B = blocks[blockIdx.y];
  Tile t;
  if (!make_tile<TL>(B, t)) return;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const ZTabS T = stage_ztab<REALZ>(tab, TAB, nz, zsm);
  __syncthreads();
  double2* fsm = zsm + ztab_slots(nz, REALZ);  // [2][FaceStage::SLOTS], then the ring
  if (!REALZ) zs2_body<0, FULL, TL>(B, t, nz, T, TAB, bufs, fsm);
  else if (B.pad_) zs2_body<2, FULL, TL>(B, t, nz, T, TAB, bufs, fsm);
  else zs2_body<1, FULL, TL>(B, t, nz, T, TAB, bufs, fsm);
}

// ===================================================================== step 5
// Per ZSEG-row segment the CTA stages R1[a][k][m0..m0+TM) and R2[b][k][l0..l0+TL) and
// forms the RHS tile with DMMA: for row j,  C[m][l] = sum_{a<KA} A1[m][a] B1[a][l]
//   + sum_{b<KA} A2[m][b] B2[b][l],  A1 = R1^T (staged), B1 = W_x[I, tile] (smem, fixed),
//   A2 = W_y[I, tile]^T (smem, fixed), B2 = R2 (staged);  KA = |I| padded to 4.
template <int TL, int NIF>
struct RankStage {
  static constexpr int TM = ZT / TL, ZSEG = 4, KA = (NIF + 3) / 4 * 4;
  static constexpr int R1S = ZSEG * KA * TM, R2S = ZSEG * KA * TL;  // per stage (double2)
  static constexpr int STAGE = R1S + R2S;
  static constexpr int RHS = ZSEG * TM * (TL + 1);                 // RHS tile [j][m][TL+1]
  static constexpr int WX = KA * TL, WY = KA * TM;                  // fixed weights
  static constexpr int FWD = 2 * STAGE + RHS + WX + WY;             // forward smem
  static constexpr int BWD = 3 * ZSEG * ZT;                         // backward ring
  static constexpr int SLOTS = FWD > BWD ? FWD : BWD;
};

template <int RT, bool FULL, int TL, int NIF>
__device__ __forceinline__ void zs3_body(const ZBlock& B, int nz, const ZTabS& T, const GSweep& G, Bufs& bufs,
                                         double2* wsm, double* minpiv_out) {
  using RS = RankStage<TL, NIF>;
  constexpr int ZSEG = RS::ZSEG, TM = RS::TM, KA = RS::KA, NSTAGE = 3;
  constexpr int CKG = 2;  // c' checkpoints every CKG segments (8 rows): c' needs no right side
  Tile t;
  {  // tiles cover this rank's global x-modes [l_begin, l_end) (all of them on one GPU)
    const int tiles_l = (G.l_end - G.l_begin + TL - 1) / TL;
    const int tl = blockIdx.x % tiles_l, tm = blockIdx.x / tiles_l;
    t.l0 = G.l_begin + tl * TL;
    t.m0 = tm * TM;
    if (t.m0 >= B.ny) return;
    t.l = t.l0 + (int)(threadIdx.x % TL);
    t.m = t.m0 + (int)(threadIdx.x / TL);
    t.active = t.l < G.l_end && t.m < B.ny;
  }
  const int r = blockIdx.z;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const double2* IF = reinterpret_cast<const double2*>(bufs.p[B_IF]);
  // wsm: union of the forward staging and the backward ring
  double2* R1s = wsm;                           // [2][ZSEG][KA][TM]
  double2* R2s = wsm + 2 * RS::R1S;             // [2][ZSEG][KA][TL]
  double2* RH = wsm + 2 * RS::STAGE;            // [ZSEG][TM][TL+1] (padded: conflict-free)
  double2* WXs = RH + RS::RHS;                  // [KA][TL]
  double2* WYs = WXs + RS::WX;                  // [KA][TM]
  const int64_t nxy = (int64_t)B.nx * B.ny;
  double2* line = reinterpret_cast<double2*>(bufs.p[B.buf]) + B.ms_off + (int64_t)r * nz * nxy +
                  (int64_t)(t.active ? t.m : 0) * B.nx + (t.active ? t.l : 0);
  const int nseg = (nz + ZSEG - 1) / ZSEG;
  const int64_t nslot = (int64_t)gridDim.x * gridDim.y * gridDim.z * ZT;
  double2* ck = ck_base(bufs);
  const int64_t RZ = (int64_t)G.R * nz;
  // fixed weights (zero beyond |I| and outside the grid); staged rows zero-filled once so
  // that entries never copied (a >= |I|, outside the grid) are finite zeros
  for (int c = threadIdx.x; c < RS::WX + RS::WY; c += ZT) {
    double2 v = make_double2(0, 0);
    if (c < RS::WX) {
      const int a = c / TL, l = t.l0 + c % TL;
      if (a < G.nifx && l < G.nx) v = TAB[G.wxi + (int64_t)a * G.nx + l];
    } else {
      const int b = (c - RS::WX) / TM, m = t.m0 + (c - RS::WX) % TM;
      if (b < G.nify && m < G.ny) v = TAB[G.wyi + (int64_t)b * G.ny + m];
    }
    WXs[c] = v;
  }
  for (int c = threadIdx.x; c < 2 * RS::STAGE; c += ZT) wsm[c] = make_double2(0, 0);
  __syncthreads();
  auto stage = [&](int sg) {
    if (sg >= 0 && sg < nseg) {
      double2* d1 = R1s + (sg & 1) * RS::R1S;
      double2* d2 = R2s + (sg & 1) * RS::R2S;
      const int k0 = sg * ZSEG;
      for (int c = threadIdx.x; c < RS::STAGE; c += ZT) {
        if (c < RS::R1S) {  // R1[a][r*nz + k][m]
          const int j = c / (KA * TM), a = (c / TM) % KA, mm = t.m0 + c % TM, k = k0 + j;
          if (a < G.nifx && mm < G.ny && (FULL || k < nz))
            cp16(d1 + c, IF + G.r1 + ((int64_t)a * RZ + (int64_t)r * nz + k) * G.ny + mm);
        } else {  // R2[b][r*nz + k][l]
          const int c2 = c - RS::R1S;
          const int j = c2 / (KA * TL), b = (c2 / TL) % KA, ll = t.l0 + c2 % TL, k = k0 + j;
          if (b < G.nify && ll < G.nx && (FULL || k < nz))
            cp16(d2 + c2, IF + G.r2 + ((int64_t)b * RZ + (int64_t)r * nz + k) * G.nx + ll);
        }
      }
    }
    cp_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int tx = threadIdx.x % TL, ty = threadIdx.x / TL;
  // warp -> row j = warp % ZSEG of the segment and (m-tile, l-tile) pairs warp / ZSEG + WPR*i
  constexpr int NT = TL / 8, MT = TM / 8, NPAIR = NT * MT, WPR = 8 / ZSEG, PPW = NPAIR / WPR;
  // 3-multiplication complex form, all pairs of the warp interleaved: 3*PPW independent
  // accumulator chains of KA/2 DMMAs each (short dependency chains, A fragments shared)
  auto rhs_tile = [&](int sg) {
    const int j = warp % ZSEG;
    const double2* a1 = R1s + (sg & 1) * RS::R1S + j * KA * TM;  // [a][m]
    const double2* b2 = R2s + (sg & 1) * RS::R2S + j * KA * TL;  // [b][l]
    double t1[PPW][2], t2[PPW][2], t3[PPW][2];
#pragma unroll
    for (int pi = 0; pi < PPW; ++pi) t1[pi][0] = t1[pi][1] = t2[pi][0] = t2[pi][1] = t3[pi][0] = t3[pi][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KA / 4; ++ks) {
      const int kk = 4 * ks + q;
#pragma unroll
      for (int pi = 0; pi < PPW; ++pi) {
        const int pr = warp / ZSEG + WPR * pi, mt = pr / NT, nt = pr % NT;
        const double2 A = a1[kk * TM + mt * 8 + g], Bv = WXs[kk * TL + nt * 8 + g];
        const double2 A2 = WYs[kk * TM + mt * 8 + g], B2 = b2[kk * TL + nt * 8 + g];
        dmma(t1[pi][0], t1[pi][1], A.x, Bv.x);
        dmma(t2[pi][0], t2[pi][1], A.y, Bv.y);
        dmma(t3[pi][0], t3[pi][1], A.x + A.y, Bv.x + Bv.y);
        dmma(t1[pi][0], t1[pi][1], A2.x, B2.x);
        dmma(t2[pi][0], t2[pi][1], A2.y, B2.y);
        dmma(t3[pi][0], t3[pi][1], A2.x + A2.y, B2.x + B2.y);
      }
    }
#pragma unroll
    for (int pi = 0; pi < PPW; ++pi) {
      const int pr = warp / ZSEG + WPR * pi, mt = pr / NT, nt = pr % NT;
      // C[m = mt*8 + g][l = nt*8 + 2q (+1)] -> the slot of thread (tx = l, ty = m)
      const int mm = mt * 8 + g, ll = nt * 8 + 2 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        RH[(j * TM + mm) * (TL + 1) + ll + h] =
            make_double2(t1[pi][h] - t2[pi][h], t3[pi][h] - t1[pi][h] - t2[pi][h]);
    }
  };
  float minpiv = 1.0f;
  const cplx s = t.active ? ld(TAB + B.lamx + t.l) + ld(TAB + B.lamy + t.m) : mk(0, 0);
  // ---- forward sweep: RHS tile per segment, d' stored in the line
  cplx cp = mk(0, 0), dp = mk(0, 0);
  stage(0);
  for (int sg = 0; sg < nseg; ++sg) {
    const int k0 = sg * ZSEG;
    stage(sg + 1);
    cp_wait<1>();
    __syncthreads();  // segment sg staged
    rhs_tile(sg);
    __syncthreads();  // RHS tile complete; staging slot sg&1 free for segment sg+2
    if (t.active) {
      if (sg % CKG == 0) ck[(int64_t)(sg / CKG) * nslot] = make_double2(cp.x, cp.y);
#pragma unroll
      for (int j = 0; j < ZSEG; ++j) {
        const int k = k0 + j;
        if (FULL || k < nz) {
          cplx a, b, c;
          double m2;
          zrow<RT>(T, k, s, a, b, c, m2);
          const double n2 = elim<RT>(a, b, c, mk(RH[(j * TM + ty) * (TL + 1) + tx]), cp, dp);
          minpiv = fminf(minpiv, __fdividef((float)n2, (float)fma(b.x, b.x, fma(b.y, b.y, m2))));
          line[(int64_t)k * nxy] = make_double2(dp.x, dp.y);  // d'
        }
      }
    }
    __syncthreads();  // RH consumed before the next tile overwrites it
  }
  cp_wait<0>();
  __threadfence_block();  // own d' stores precede the cp.async re-reads
  __syncthreads();        // the forward staging area becomes the backward ring
  const Ring<ZSEG, NSTAGE, FULL> ring{wsm, line, nxy, nz, t.active};
#pragma unroll
  for (int qq = 0; qq < NSTAGE - 1; ++qq) ring.issue(nseg - 1 - qq);
  cplx x = mk(0, 0);
  const int ngrp = (nseg + CKG - 1) / CKG;
  double2 nc = ck[(int64_t)(ngrp - 1) * nslot];
  for (int gi = ngrp - 1; gi >= 0; --gi) {
    // c' of the group's rows recomputed from its checkpoint (no right side needed)
    cplx cs[CKG * ZSEG];
    cplx cc = mk(nc);
    if (gi > 0) nc = ck[(int64_t)(gi - 1) * nslot];
    if (t.active) {
#pragma unroll
      for (int j = 0; j < CKG * ZSEG; ++j) {
        const int k = gi * CKG * ZSEG + j;
        if (FULL || k < nz) {
          cplx a, b, c;
          double m2;
          zrow<RT>(T, k, s, a, b, c, m2);
          elim_c<RT>(a, b, c, cc);
        }
        cs[j] = cc;
      }
    }
#pragma unroll
    for (int q = CKG - 1; q >= 0; --q) {
      const int sg = gi * CKG + q;
      if (sg >= nseg) continue;  // uniform: the last group may be short
      const int k0 = sg * ZSEG;
      ring.issue(sg - (NSTAGE - 1));
      cp_wait<NSTAGE - 1>();
      if (!t.active) continue;
      double2* lp = line + (int64_t)k0 * nxy;
#pragma unroll
      for (int j = ZSEG - 1; j >= 0; --j) {
        if (FULL || k0 + j < nz) {
          x = backsub<RT>(ring.get(sg, j), cs[q * ZSEG + j], x);
          lp[j * nxy] = make_double2(x.x, x.y);
        }
      }
    }
  }
  cp_wait<0>();
  commit_minpiv(minpiv, minpiv_out);
}


template <bool REALZ, int TL, int NIF, bool FULL>
__global__ void __launch_bounds__(ZT, 3) k_zs3(const ZBlock* __restrict__ blocks, int nz, ZTab tab, GSweep G,
                                               Bufs bufs, double* minpiv_out) {
  extern __shared__ __align__(16) double2 zsm[];
  const ZBlock B = blocks[blockIdx.y];
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const ZTabS T = stage_ztab<REALZ>(tab, TAB, nz, zsm);  // barrier inside the body
  double2* wsm = zsm + ztab_slots(nz, REALZ);
  if (!REALZ) zs3_body<0, FULL, TL, NIF>(B, nz, T, G, bufs, wsm, minpiv_out);
  else if (B.pad_) zs3_body<2, FULL, TL, NIF>(B, nz, T, G, bufs, wsm, minpiv_out);
  else zs3_body<1, FULL, TL, NIF>(B, nz, T, G, bufs, wsm, minpiv_out);
}

// ===================================================================== step 2, warp per line
// k_zsw: the step-2 systems T_lm v~_lm = f~_lm with ONE read and ONE write of every mode-space
// value (k_zs1 reads the right side twice: its per-thread lines do not fit on chip, so the
// backward sweep re-reads them).  A warp solves one z-line held in its registers, Q = 32-row
// chunks per lane ("partition" form of Thomas, the warp-shuffle PCR/Thomas hybrid of the
// north_star):
//   1. each lane eliminates the interior rows of its chunk (Thomas, unpivoted like k_zs1,
//      reading R15): interior x = y - L X_{t-1} - R X_t, with X_t the lane's last row (the
//      separator) and y, L, R the chunk solves for the right side and the two coupling spikes;
//   2. the separators obey a 32-row tridiagonal system (lane t: row X_t, coupled to X_{t-1}
//      and X_{t+1} through the neighbours' spikes), solved by parallel cyclic reduction over the
//      lanes with shuffles (5 steps);
//   3. every lane forms its interior values from X_{t-1} and X_t.
// Mode tiles (8 consecutive l at one m, all N_z rows: 128-B rows) are staged by coalesced 16-B
// cp.async copies, NBUF-buffered in a persistent loop (the next tiles land while the current one
// is solved), and stored back by coalesced rows.  Rows are padded to 9 units and Q is odd, so
// the 8 lanes of a shared-memory phase (rows tQ + j, t = 0..7) hit 8 different bank groups.
// (A first version staged each 128-B row with a cp.async.bulk copy on an mbarrier: correct and
// single-read, but ~10x slower: 512 tiny bulk operations per tile serialise on the copy engine.)
constexpr int ZW_WARPS = 8, ZW_TL = 8;  // lines (l) per tile = warps per CTA

template <int Q>
struct ZwTile {  // 16-B units of one tile buffer: rows of 8 complex + 1 pad unit (odd stride)
  static constexpr int W = ZW_TL + 1;
  static constexpr int UNITS = W * 32 * Q;
  __device__ static __forceinline__ int row(int k) { return W * k; }
};

__device__ __forceinline__ cplx shfl_c(cplx v, int src) {
  return mk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double shfl_c(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
// coefficient arithmetic: TC = double for real systems (RT 2: real table and real shift: the
// pivots, c' and both spikes are real), cplx otherwise; data (right side, y, X) always cplx
__device__ __forceinline__ cplx cm(double a, cplx b) { return mk(a * b.x, a * b.y); }
__device__ __forceinline__ cplx cm(cplx a, cplx b) { return a * b; }
__device__ __forceinline__ double cm(double a, double b) { return a * b; }
__device__ __forceinline__ double tc_n2(double a) { return a * a; }
__device__ __forceinline__ double tc_n2(cplx a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double tc_abs1(double a) { return fabs(a); }
__device__ __forceinline__ double tc_abs1(cplx a) { return cabs1(a); }
__device__ __forceinline__ double tc_inv(double r) { return fast_rcp(r); }
__device__ __forceinline__ cplx tc_inv(cplx r) {
  const double in = fast_rcp(fma(r.x, r.x, r.y * r.y));
  return mk(r.x * in, -r.y * in);
}
__device__ __forceinline__ double tc_neg(double a) { return -a; }
__device__ __forceinline__ cplx tc_neg(cplx a) { return mk(-a.x, -a.y); }
__device__ __forceinline__ double tc_zero(double) { return 0.0; }
__device__ __forceinline__ cplx tc_zero(cplx) { return mk(0, 0); }
__device__ __forceinline__ double tc_one(double) { return 1.0; }
__device__ __forceinline__ cplx tc_one(cplx) { return mk(1, 0); }

// the row coefficients of T_lm (zrow) in the coefficient type
template <int RT, class TC>
__device__ __forceinline__ void zrow_tc(const ZTabS& T, int k, int nz, cplx s, TC& a, TC& b, TC& c, double& m2) {
  if (k >= nz) {  // padding rows: identity, decoupled (row nz-1 has c = 0)
    a = tc_zero(a); b = tc_one(b); c = tc_zero(c); m2 = 0;
    return;
  }
  cplx ac, bc, cc;
  zrow<RT>(T, k, s, ac, bc, cc, m2);
  if constexpr (RT == 2) { a = ac.x; b = bc.x; c = cc.x; }
  else { a = ac; b = bc; c = cc; }
}

// one line: lane t owns rows tQ .. tQ+Q-1 (values in x[], from and back into the tile)
template <int RT, int Q>
__device__ __forceinline__ float zsw_line(const ZTabS& T, int nz, cplx s, cplx (&x)[Q]) {
  using TC = typename std::conditional<RT == 2, double, cplx>::type;
  const int t = threadIdx.x & 31;
  const int k0 = t * Q;
  const int J = t < 31 ? Q - 1 : Q;  // interior rows (the last lane has no separator)
  float minpiv = 1.0f;
  // ---- 1. interior chunk: Thomas forward elimination (pivot r, c' = c / r) with three right
  // sides: the data (y, kept in x[]), the spike of X_{t-1} (a_0 e_0: L) and of X_t
  // (c_{J-1} e_{J-1}: R, whose forward value is just c'_{J-1})
  TC cp[Q], Lv[Q], Rv[Q];
  {
    TC cprev = tc_zero(TC{}), lprev = tc_zero(TC{});
    cplx dprev = mk(0, 0);
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      if (j < J) {
        TC a, b, c;
        double m2;
        zrow_tc<RT>(T, k0 + j, nz, s, a, b, c, m2);
        const TC r = j == 0 ? b : b - cm(a, cprev);
        const TC inv = tc_inv(r);
        const double bn = tc_abs1(b);
        minpiv = fminf(minpiv, __fdividef((float)tc_n2(r), (float)fma(bn, bn, m2) + 1e-30f));
        cp[j] = cm(c, inv);
        x[j] = cm(inv, j == 0 ? x[j] : x[j] - cm(a, dprev));
        Lv[j] = j == 0 ? cm(a, inv) : tc_neg(cm(cm(a, lprev), inv));
        Rv[j] = tc_zero(TC{});
        cprev = cp[j]; dprev = x[j]; lprev = Lv[j];
      }
    }
    if (J > 0) Rv[J - 1] = cp[J - 1];
    // back substitution of the three right sides
#pragma unroll
    for (int j = Q - 2; j >= 0; --j) {
      if (j < J - 1) {
        x[j] = x[j] - cm(cp[j], x[j + 1]);
        Lv[j] = Lv[j] - cm(cp[j], Lv[j + 1]);
        Rv[j] = tc_neg(cm(cp[j], Rv[j + 1]));
      }
    }
  }
  // ---- 2. separator system (lane t < 31: unknown X_t = row tQ + Q - 1), PCR over the lanes
  const int up = (t + 1) & 31;
  const cplx yf = shfl_c(x[0], up);
  const TC Lf = shfl_c(Lv[0], up), Rf = shfl_c(Rv[0], up);
  TC A = tc_zero(TC{}), Bc = tc_one(TC{}), C = tc_zero(TC{});
  cplx D = mk(0, 0);
  if (t < 31) {
    TC a, b, c;
    double m2;
    zrow_tc<RT>(T, k0 + Q - 1, nz, s, a, b, c, m2);
    // x_{k-1} = y_{Q-2} - L_{Q-2} X_{t-1} - R_{Q-2} X_t ;  x_{k+1} = yf - Lf X_t - Rf X_{t+1}
    A = tc_neg(cm(a, Lv[Q - 2]));
    Bc = b - cm(a, Rv[Q - 2]) - cm(c, Lf);
    C = tc_neg(cm(c, Rf));
    D = x[Q - 1] - cm(a, x[Q - 2]) - cm(c, yf);
  }
  const double bnorm = tc_abs1(A) + tc_abs1(Bc) + tc_abs1(C);
#pragma unroll
  for (int dl = 1; dl < 32; dl <<= 1) {
    const int lo = t - dl, hi = t + dl;
    const TC Al = shfl_c(A, lo & 31), Bl = shfl_c(Bc, lo & 31), Cl = shfl_c(C, lo & 31);
    const TC Ah = shfl_c(A, hi & 31), Bh = shfl_c(Bc, hi & 31), Ch = shfl_c(C, hi & 31);
    const cplx Dl = shfl_c(D, lo & 31), Dh = shfl_c(D, hi & 31);
    const TC al = lo >= 0 ? tc_neg(cm(A, tc_inv(Bl))) : tc_zero(TC{});
    const TC ga = hi < 32 ? tc_neg(cm(C, tc_inv(Bh))) : tc_zero(TC{});
    const TC An = cm(al, Al), Cn = cm(ga, Ch);
    Bc = Bc + cm(al, Cl) + cm(ga, Ah);
    D = D + cm(al, Dl) + cm(ga, Dh);
    A = An;
    C = Cn;
  }
  const cplx X = t < 31 ? cm(tc_inv(Bc), D) : mk(0, 0);
  if (t < 31 && bnorm > 0) {
    const float q = (float)(tc_abs1(Bc) / bnorm);
    minpiv = fminf(minpiv, q * q);
  }
  const cplx Xs = shfl_c(X, (t - 1) & 31);
  const cplx Xl = t > 0 ? Xs : mk(0, 0);
  // ---- 3. interior values
#pragma unroll
  for (int j = 0; j < Q; ++j)
    if (j < J) x[j] = x[j] - cm(Lv[j], Xl) - cm(Rv[j], X);
  if (t < 31) x[Q - 1] = X;
  return minpiv;
}

// NBUF tile buffers: NBUF - 1 tiles in flight (cp.async) while one is solved.  Persistent grid
// over the flattened (block, rhs, tile) items of one system class: every SM busy to the end.
template <int RT, int Q, int NBUF>
__global__ void __launch_bounds__(ZW_WARPS * 32, RT == 2 ? 2 : 1) k_zsw(const ZBlock* __restrict__ blocks,
                                                                      const int* __restrict__ order, int nblocks,
                                                                      int R, int tiles_per, int nz, ZTab tab,
                                                                      Bufs bufs, double* minpiv_out) {
  constexpr bool REALZ = RT >= 1;
  static_assert(Q % 2 == 1, "odd rows per lane: conflict-free chunk reads with the 9-unit row stride");
  extern __shared__ __align__(16) double2 zsm[];
  using TT = ZwTile<Q>;
  const double2* TAB = reinterpret_cast<const double2*>(bufs.p[B_TAB]);
  const ZTabS T = stage_ztab<REALZ>(tab, TAB, nz, zsm);
  double2* tiles = zsm + ((ztab_slots(nz, REALZ) + 7) & ~7);  // tile buffers after the z table
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t items = (int64_t)nblocks * R * tiles_per;
  // item -> block, rhs, tile (m-major, 8-wide l tiles); false for the padding items of blocks
  // smaller than the largest one
  struct Item { const ZBlock* B; double2* src; int nv, l, m; };
  auto locate = [&](int64_t it, Item& I) -> bool {
    const int tile = (int)(it % tiles_per);
    const int64_t br = it / tiles_per;
    const int r = (int)(br % R), b = (int)(br / R);
    const ZBlock& Bk = blocks[order[b]];
    const int tiles_l = (Bk.nx + ZW_TL - 1) / ZW_TL;
    const int m = tile / tiles_l, l0 = (tile - m * tiles_l) * ZW_TL;
    if (m >= Bk.ny) return false;
    const int64_t nxy = (int64_t)Bk.nx * Bk.ny;
    I.B = &Bk;
    I.nv = min(ZW_TL, Bk.nx - l0);
    I.l = l0;
    I.m = m;
    I.src = reinterpret_cast<double2*>(bufs.p[Bk.buf]) + Bk.ms_off + (int64_t)r * nz * nxy + (int64_t)m * Bk.nx + l0;
    return true;
  };
  // coalesced 16-B cp.async loads of an item into buffer `bf`: a warp covers four 128-B rows
  auto issue = [&](int64_t it, int bf) {
    Item I;
    if (it < items && locate(it, I)) {
      const int64_t nxy = (int64_t)I.B->nx * I.B->ny;
      double2* dst = tiles + bf * TT::UNITS;
      for (int idx = threadIdx.x; idx < nz * ZW_TL; idx += ZW_WARPS * 32) {
        const int k = idx >> 3, w = idx & 7;
        if (w < I.nv) cp16(dst + TT::row(k) + w, I.src + (int64_t)k * nxy + w);
      }
    }
    cp_commit();
  };
  float minpiv = 1.0f;
  const int64_t it0 = blockIdx.x, G = gridDim.x;
#pragma unroll
  for (int q = 0; q < NBUF - 1; ++q) issue(it0 + q * G, q);
  int n = 0;
  for (int64_t it = it0; it < items; it += G, ++n) {
    const int bf = n % NBUF;
    __syncthreads();  // buffer (n - 1) % NBUF fully stored by the previous iteration
    issue(it + (NBUF - 1) * G, (n + NBUF - 1) % NBUF);
    cp_wait<NBUF - 1>();
    __syncthreads();  // item n visible to every warp
    Item I;
    if (!locate(it, I)) continue;
    const int64_t nxy = (int64_t)I.B->nx * I.B->ny;
    double2* tb = tiles + bf * TT::UNITS;
    if (warp < I.nv) {
      const cplx s = ld(TAB + I.B->lamx + I.l + warp) + ld(TAB + I.B->lamy + I.m);
      cplx x[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const int k = lane * Q + j;
        x[j] = k < nz ? mk(tb[TT::row(k) + warp]) : mk(0, 0);
      }
      minpiv = fminf(minpiv, zsw_line<RT, Q>(T, nz, s, x));
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const int k = lane * Q + j;
        if (k < nz) tb[TT::row(k) + warp] = make_double2(x[j].x, x[j].y);
      }
    }
    __syncthreads();  // the solved tile back in shared memory
    for (int idx = threadIdx.x; idx < nz * ZW_TL; idx += ZW_WARPS * 32) {
      const int k = idx >> 3, w = idx & 7;
      if (w < I.nv) I.src[(int64_t)k * nxy + w] = tb[TT::row(k) + w];
    }
  }
  cp_wait<0>();
  commit_minpiv(minpiv, minpiv_out);
}

template <int RT, int Q>
cudaError_t zsw_launch(const ZBlock* b, const int* order, int nblocks, int max_nx, int max_ny, int R, int nz, ZTab tab,
                       const Bufs& bufs, double* mp, cudaStream_t st) {
  constexpr bool REALZ = RT >= 1;
  // 2 CTAs/SM (real: 128 registers) or 1 with 2 tiles in flight; 2 buffers for the longest lines
  // (Q = 17: 78 KB per tile)
  constexpr int NBUF = (RT == 2 || Q > 9) ? 2 : 3;
  const size_t sm = (size_t)(((ztab_slots(nz, REALZ) + 7) & ~7) + NBUF * ZwTile<Q>::UNITS) * sizeof(double2);
  auto kern = k_zsw<RT, Q, NBUF>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, ZW_WARPS * 32, sm)) != cudaSuccess) return e;
  const int tiles_per = ((max_nx + ZW_TL - 1) / ZW_TL) * max_ny;
  const int64_t items = (int64_t)nblocks * R * tiles_per;
  const int64_t grid = std::min<int64_t>(items, (int64_t)std::max(1, per) * sms);
  kern<<<(unsigned)grid, ZW_WARPS * 32, sm, st>>>(b, order, nblocks, R, tiles_per, nz, tab, bufs, mp);
  return cudaGetLastError();
}

template <int RT>
cudaError_t zsw_dispatch(const ZBlock* b, const int* order, int nblocks, int max_nx, int max_ny, int R, int nz,
                         ZTab tab, const Bufs& bufs, double* mp, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  if (nz <= 96) return zsw_launch<RT, 3>(b, order, nblocks, max_nx, max_ny, R, nz, tab, bufs, mp, st);
  if (nz <= 160) return zsw_launch<RT, 5>(b, order, nblocks, max_nx, max_ny, R, nz, tab, bufs, mp, st);
  if (nz <= 288) return zsw_launch<RT, 9>(b, order, nblocks, max_nx, max_ny, R, nz, tab, bufs, mp, st);
  return zsw_launch<RT, 17>(b, order, nblocks, max_nx, max_ny, R, nz, tab, bufs, mp, st);
}

// ===================================================================== launch
int tile_l(int mode, int max_nx, int nif) {
  if (mode == 3 && nif > 8) return 16;  // keeps the 16-row staging of k_zs3 within 2 CTAs/SM
  if (mode == 2) return 16;             // step 6: 16 x 16 tiles stage fewer face rows (measured 2.60 -> 2.52 ms at C4)
  return max_nx > 16 ? 32 : 16;
}

dim3 zs_grid(int nblocks, int max_nx, int max_ny, int R, int tl) {
  const int tm = ZT / tl;
  const int tiles = ((max_nx + tl - 1) / tl) * ((max_ny + tm - 1) / tm);
  return dim3((unsigned)tiles, (unsigned)nblocks, (unsigned)R);
}

template <class K>
cudaError_t prep(K kern, size_t sm) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

// experiment knob (tools/zs_occupancy.sh): extra dynamic shared memory per CTA of the step-2 /
// step-6 solvers, to force fewer CTAs per SM (fewer lines in flight: the backward-sweep re-read
// of k_zs1 then hits L2).  0 unless LFDS_ZS_PAD1 / LFDS_ZS_PAD2 is set.
size_t zs_pad(int mode) {
  static long p1 = -1, p2 = -1;
  if (p1 < 0) {
    const char* a = getenv("LFDS_ZS_PAD1");
    const char* b = getenv("LFDS_ZS_PAD2");
    p1 = a ? atol(a) : 0;
    p2 = b ? atol(b) : 0;
  }
  return (size_t)(mode == 1 ? p1 : mode == 2 ? p2 : 0);
}

template <bool REALZ, int TL, bool FULL>
cudaError_t launch_tl(int mode, dim3 grid, cudaStream_t st, const ZBlock* b, int nz, ZTab tab, const GSweep& g,
                      const Bufs& bufs, double* mp) {
  const size_t zt = (size_t)ztab_slots(nz, REALZ) * sizeof(double2);
  cudaError_t e;
  if (mode == 1) {
    const size_t sm = zt + (size_t)3 * 8 * ZT * sizeof(double2) + zs_pad(1);
    if ((e = prep(k_zs1<REALZ, TL, FULL>, sm)) != cudaSuccess) return e;
    k_zs1<REALZ, TL, FULL><<<grid, ZT, sm, st>>>(b, nz, tab, bufs, mp);
  } else if (mode == 2) {
    const size_t sm = zt + (size_t)(2 * FaceStage<TL, 16>::SLOTS + 2 * 8 * ZT) * sizeof(double2) + zs_pad(2);
    if ((e = prep(k_zs2<REALZ, TL, FULL>, sm)) != cudaSuccess) return e;
    k_zs2<REALZ, TL, FULL><<<grid, ZT, sm, st>>>(b, nz, tab, bufs);
  } else {
    const int nif = g.nifx > g.nify ? g.nifx : g.nify;
#define Z3(N)                                                                     \
  {                                                                               \
    const size_t sm = zt + (size_t)RankStage<TL, N>::SLOTS * sizeof(double2);     \
    if ((e = prep(k_zs3<REALZ, TL, N, FULL>, sm)) != cudaSuccess) return e;       \
    k_zs3<REALZ, TL, N, FULL><<<grid, ZT, sm, st>>>(b, nz, tab, g, bufs, mp);     \
  }
    if (nif <= 4) Z3(4)
    else if (nif <= 8) Z3(8)
    else if (nif <= 16) Z3(16)
    else return cudaErrorInvalidValue;
#undef Z3
  }
  return cudaGetLastError();
}

template <bool REALZ, int TL>
cudaError_t launch_full(int mode, dim3 grid, cudaStream_t st, const ZBlock* b, int nz, ZTab tab, const GSweep& g,
                        const Bufs& bufs, double* mp) {
  // no ragged tail: 8-row segments (steps 2, 6) and 8-row checkpoint groups (step 5)
  const bool full = nz % 8 == 0;
  return full ? launch_tl<REALZ, TL, true>(mode, grid, st, b, nz, tab, g, bufs, mp)
              : launch_tl<REALZ, TL, false>(mode, grid, st, b, nz, tab, g, bufs, mp);
}

}  // namespace

size_t zsolve_checkpoint_bytes(int nblocks, int max_nx, int max_ny, int R, int nz) {
  // steps 2/6: (c', d') every 8 rows; step 5: c' every 4 rows; either tile shape
  size_t slots = 0;
  for (int tl : {16, 32}) {
    const dim3 g = zs_grid(nblocks, max_nx, max_ny, R, tl);
    slots = std::max(slots, (size_t)g.x * g.y * g.z * ZT);
  }
  const size_t per = (size_t)((nz + 3) / 4 + 1);
  return slots * per * sizeof(double2);
}

cudaError_t launch_zsolve(int mode, const ZBlock* d_blocks, int nblocks, int max_nx, int max_ny, int R, int nz,
                          ZTab tab, int64_t sig_off, const GSweep* g, const Bufs& bufs, double* d_minpiv,
                          cudaStream_t st, bool realz) {
  if (R > 65535 || nblocks > 65535) return cudaErrorInvalidValue;
  GSweep G{};
  if (g) G = *g;
  const int tl = tile_l(mode, max_nx, G.nifx > G.nify ? G.nifx : G.nify);
  const dim3 grid = zs_grid(nblocks, mode == 3 ? G.l_end - G.l_begin : max_nx, max_ny, R, tl);
  if (grid.x == 0) return cudaSuccess;
  (void)sig_off;
  if (realz) return tl == 32 ? launch_full<true, 32>(mode, grid, st, d_blocks, nz, tab, G, bufs, d_minpiv)
                             : launch_full<true, 16>(mode, grid, st, d_blocks, nz, tab, G, bufs, d_minpiv);
  return tl == 32 ? launch_full<false, 32>(mode, grid, st, d_blocks, nz, tab, G, bufs, d_minpiv)
                  : launch_full<false, 16>(mode, grid, st, d_blocks, nz, tab, G, bufs, d_minpiv);
}

bool zsw_supported(int nz) { return nz >= 2 && nz <= 544; }

cudaError_t launch_zsw(const ZBlock* d_blocks, const int* d_order, const int counts[3], int max_nx, int max_ny, int R,
                       int nz, ZTab tab, const Bufs& bufs, double* d_minpiv, cudaStream_t st) {
  if (R > 65535) return cudaErrorInvalidValue;
  cudaError_t e;
  // d_order lists the blocks by class: complex tables (RT 0), real tables with a complex shift
  // (RT 1), real tables and shift (RT 2)
  if ((e = zsw_dispatch<0>(d_blocks, d_order, counts[0], max_nx, max_ny, R, nz, tab, bufs, d_minpiv, st))) return e;
  if ((e = zsw_dispatch<1>(d_blocks, d_order + counts[0], counts[1], max_nx, max_ny, R, nz, tab, bufs, d_minpiv, st)))
    return e;
  return zsw_dispatch<2>(d_blocks, d_order + counts[0] + counts[1], counts[2], max_nx, max_ny, R, nz, tab, bufs,
                         d_minpiv, st);
}

}  // namespace lfds
