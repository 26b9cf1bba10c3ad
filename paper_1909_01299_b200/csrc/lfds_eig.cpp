// Host eigensolver for the 1D pencils (A_d, M_d) of PAPER.md:45-46 and :55 (per-block and
// global generalized eigenproblems A W = M W Lambda with homogeneous Dirichlet ends).
//
// Written for this library (no LAPACK on the host side of the C library):
//  * symmetrise S = M^{-1/2} A M^{-1/2} (principal complex square root): complex symmetric
//    tridiagonal, so S = V Lambda V^T with V^T V = I (transpose, reading R4 of DESIGN.md);
//  * mirror-symmetric (palindromic) step sequences are split into the even and odd
//    invariant subspaces first (their eigenvalues interleave and are numerically
//    degenerate under PML otherwise);
//  * eigenvalues by the implicit QL iteration with complex "rotations" (c^2 + s^2 = 1),
//    eigenvectors by inverse iteration with a partially pivoted tridiagonal LU, both in
//    80-bit long double; clusters are re-biorthogonalised in the bilinear form;
//  * uniform real steps use the closed form W_il = sqrt(2/(h(n+1))) sin(pi i l/(n+1)),
//    lambda_l = -(4/h^2) sin^2(pi l / (2(n+1)))  (the 'Fourier transform' of PAPER.md:47, :75).
#include "lfds_eig.h"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <numeric>

namespace lfds {

using lc = std::complex<long double>;
static inline long double abs1(lc z) { return std::fabs(z.real()) + std::fabs(z.imag()); }

// implicit QL on (d, e), e[i] couples i and i+1; returns false on non-convergence/breakdown.
// The textbook implicit-shift QL iteration (the EISPACK tql1 / Numerical Recipes tqli loop
// structure), here complexified for complex-symmetric pencils and run in long double.
static bool ql_values(std::vector<lc>& d, std::vector<lc> e) {
  const int n = (int)d.size();
  if (n <= 1) return true;
  e.resize(n);
  e[n - 1] = 0;
  const long double eps = LDBL_EPSILON;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    for (;;) {
      int m = l;
      for (; m < n - 1; ++m) {
        long double dd = abs1(d[m]) + abs1(d[m + 1]);
        if (abs1(e[m]) <= eps * dd) break;
      }
      if (m == l) break;
      if (++iter > 200) return false;
      lc g = (d[l + 1] - d[l]) / (2.0L * e[l]);
      lc r = std::sqrt(g * g + lc(1.0L));
      lc gp = (std::abs(g + r) >= std::abs(g - r)) ? g + r : g - r;
      if (gp == lc(0)) return false;
      g = d[m] - d[l] + e[l] / gp;
      lc s = 1, c = 1, p = 0;
      bool early = false;
      for (int i = m - 1; i >= l; --i) {
        lc f = s * e[i], b = c * e[i];
        r = std::sqrt(f * f + g * g);
        e[i + 1] = r;
        if (abs1(r) <= 1e-300L * (abs1(f) + abs1(g)) || r == lc(0)) {
          if (abs1(f) + abs1(g) == 0) {
            d[i + 1] -= p;
            e[m] = 0;
            early = true;
            break;
          }
          return false;  // isotropic rotation: breakdown of the complex-symmetric QL
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0L * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
      }
      if (early) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0;
    }
  }
  return true;
}

// one eigenvector of the tridiagonal (d, e) at eigenvalue mu by inverse iteration; the shifted
// matrix is factored by LU with partial pivoting in the dl / d / du / du2 band layout of LAPACK's
// zgttrf (the standard algorithm, written out here in long double).
static void inverse_iteration(const std::vector<lc>& d, const std::vector<lc>& e, lc mu, long double snorm,
                              std::vector<lc>& x, int seed, int iters, bool fresh) {
  const int n = (int)d.size();
  std::vector<lc> dl(n), dd(n), du(n), du2(n);
  std::vector<int> piv(n);
  for (int i = 0; i < n; ++i) dd[i] = d[i] - mu;
  for (int i = 0; i + 1 < n; ++i) dl[i] = du[i] = e[i];
  const long double tiny = LDBL_EPSILON * (snorm > 0 ? snorm : 1.0L);
  for (int i = 0; i + 1 < n; ++i) {
    du2[i] = 0;
    if (abs1(dd[i]) >= abs1(dl[i])) {
      if (abs1(dd[i]) < tiny) dd[i] = tiny;
      lc fact = dl[i] / dd[i];
      dl[i] = fact;
      dd[i + 1] -= fact * du[i];
      piv[i] = i;
    } else {
      lc fact = dd[i] / dl[i];
      dd[i] = dl[i];
      dl[i] = fact;
      lc tmp = du[i];
      du[i] = dd[i + 1];
      dd[i + 1] = tmp - fact * dd[i + 1];
      if (i + 2 < n) {
        du2[i] = du[i + 1];
        du[i + 1] = -fact * du[i + 1];
      }
      piv[i] = i + 1;
    }
  }
  if (abs1(dd[n - 1]) < tiny) dd[n - 1] = tiny;
  if (fresh) {  // deterministic start vector
    x.assign(n, lc(0));
    unsigned s = 2654435761u * (unsigned)(seed + 1);
    for (int i = 0; i < n; ++i) {
      s = s * 1664525u + 1013904223u;
      x[i] = lc(0.5L + (long double)(s >> 8) / 16777216.0L, 0.0L);
    }
  }
  for (int it = 0; it < iters; ++it) {
    // forward: L with row interchanges
    for (int i = 0; i + 1 < n; ++i) {
      if (piv[i] == i) {
        x[i + 1] -= dl[i] * x[i];
      } else {
        lc t = x[i];
        x[i] = x[i + 1];
        x[i + 1] = t - dl[i] * x[i];
      }
    }
    // back: U with du, du2
    x[n - 1] /= dd[n - 1];
    if (n > 1) x[n - 2] = (x[n - 2] - du[n - 2] * x[n - 1]) / dd[n - 2];
    for (int i = n - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / dd[i];
    long double mx = 0;
    for (int i = 0; i < n; ++i) mx = std::max(mx, abs1(x[i]));
    if (mx == 0) mx = 1;
    for (int i = 0; i < n; ++i) x[i] /= mx;
  }
}

// p(mu)/p'(mu) for p = det(S - mu I) through the ratios d_k = p_k / p_{k-1}
static lc newton_ratio(const std::vector<lc>& d, const std::vector<lc>& e, lc mu, long double snorm) {
  const int n = (int)d.size();
  const long double tiny = 1e-30L * (snorm > 0 ? snorm : 1.0L);
  lc q = d[0] - mu, qp = -1;
  if (abs1(q) < tiny) q = tiny;
  lc acc = qp / q;
  for (int k = 1; k < n; ++k) {
    lc e2 = e[k - 1] * e[k - 1];
    lc qn = (d[k] - mu) - e2 / q;
    lc qpn = lc(-1) + e2 * qp / (q * q);
    if (abs1(qn) < tiny) qn = tiny;
    q = qn;
    qp = qpn;
    acc += qp / q;
  }
  return lc(1) / acc;
}

static bool aberth_polish(const std::vector<lc>& d, const std::vector<lc>& e, std::vector<lc>& lam,
                          long double snorm) {
  const int n = (int)lam.size();
  if (n <= 1) {
    if (n == 1) lam[0] = d[0];
    return true;
  }
  const long double tol = 8 * LDBL_EPSILON * (snorm > 0 ? snorm : 1.0L);
  // a root is done when its correction is at the long-double level, or when it has
  // stagnated at the noise floor of an ill-conditioned (non-normal) eigenvalue
  const long double floor_tol = 1e-9L * (snorm > 0 ? snorm : 1.0L);
  std::vector<char> done(n, 0);
  std::vector<long double> prev(n, 1e300L);
  for (int sweep = 0; sweep < 200; ++sweep) {
    int active = 0;
    for (int i = 0; i < n; ++i) {
      if (done[i]) continue;
      lc N = newton_ratio(d, e, lam[i], snorm);
      lc S = 0;
      for (int j = 0; j < n; ++j)
        if (j != i) S += lc(1) / (lam[i] - lam[j]);
      lc w = N / (lc(1) - N * S);
      const long double aw = std::abs(w);
      if (aw <= tol || (sweep > 4 && aw >= 0.5L * prev[i] && aw < floor_tol)) {
        if (aw < prev[i]) lam[i] -= w;
        done[i] = 1;
        continue;
      }
      lam[i] -= w;
      prev[i] = aw;
      ++active;
    }
    if (!active) return true;
  }
  return false;
}

// eigenpairs of the complex symmetric tridiagonal (d, e): V column-major V[i + n*j]
static bool tridiag_eig(const std::vector<lc>& d, const std::vector<lc>& e, std::vector<lc>& lam,
                        std::vector<lc>& V) {
  const int n = (int)d.size();
  lam = d;
  if (!ql_values(lam, e)) {
    // QL broke down (isotropic rotation) or stalled: seed Aberth from the spectrum of the
    // real part instead (a real symmetric tridiagonal, for which QL cannot break down)
    std::vector<lc> dr(n), er(e.size());
    for (int i = 0; i < n; ++i) dr[i] = lc(d[i].real(), 0);
    for (size_t i = 0; i < e.size(); ++i) er[i] = lc(e[i].real(), 0);
    lam = dr;
    if (!ql_values(lam, er)) lam = d;
    for (int i = 0; i < n; ++i) lam[i] += lc(0, 1e-3L * (1 + i % 7)) * (std::abs(lam[i]) + 1e-3L);
  }
  std::sort(lam.begin(), lam.end(), [](lc a, lc b) {
    return a.real() < b.real() || (a.real() == b.real() && a.imag() < b.imag());
  });
  long double snorm = 0;
  for (int i = 0; i < n; ++i) snorm = std::max(snorm, abs1(d[i]) + (i ? abs1(e[i - 1]) : 0) + (i + 1 < n ? abs1(e[i]) : 0));
  V.assign((size_t)n * n, lc(0));
  std::vector<lc> x;
  // The complex-symmetric QL uses non-unitary rotations and loses digits on long
  // non-normal (PML) pencils, so its eigenvalues only seed a simultaneous Aberth-Ehrlich
  // iteration on det(S - mu I), evaluated by the three-term recurrence: every root is
  // polished to long-double accuracy and no two estimates can settle on the same root.
  if (!aberth_polish(d, e, lam, snorm)) return false;  // caller reports EEIG
  std::sort(lam.begin(), lam.end(), [](lc a, lc b) {
    return a.real() < b.real() || (a.real() == b.real() && a.imag() < b.imag());
  });
  for (int j = 0; j < n; ++j) {
    inverse_iteration(d, e, lam[j], snorm, x, j, 3, true);
    lc nn = 0;
    for (int i = 0; i < n; ++i) nn += x[i] * x[i];
    lc sc = lc(1) / std::sqrt(nn);
    for (int i = 0; i < n; ++i) V[i + (size_t)n * j] = x[i] * sc;
  }
  // re-biorthogonalise clusters of close eigenvalues (bilinear Gram-Schmidt, two passes)
  const long double ctol = 1e-7L * (snorm > 0 ? snorm : 1.0L);
  for (int j = 1; j < n; ++j) {
    for (int pass = 0; pass < 2; ++pass) {
      bool touched = false;
      for (int i = j - 1; i >= 0 && std::abs(lam[j] - lam[i]) <= ctol * 1e3L; --i) {
        if (std::abs(lam[j] - lam[i]) > ctol) continue;
        lc dot = 0;
        for (int q = 0; q < n; ++q) dot += V[q + (size_t)n * i] * V[q + (size_t)n * j];
        for (int q = 0; q < n; ++q) V[q + (size_t)n * j] -= dot * V[q + (size_t)n * i];
        touched = true;
      }
      if (!touched) break;
      lc nn = 0;
      for (int q = 0; q < n; ++q) nn += V[q + (size_t)n * j] * V[q + (size_t)n * j];
      lc sc = lc(1) / std::sqrt(nn);
      for (int q = 0; q < n; ++q) V[q + (size_t)n * j] *= sc;
    }
  }
  return true;
}

bool pencil_basis(const std::vector<zc>& h, Basis& B, std::string& err, const std::vector<zc>* mass) {
  const int n = (int)h.size() - 1;
  if (mass && (int)mass->size() != n) {
    err = "mass size";
    return false;
  }
  auto hhat = [&](int i) -> lc {
    if (mass) return lc((*mass)[i].real(), (*mass)[i].imag());
    return 0.5L * (lc(h[i].real(), h[i].imag()) + lc(h[i + 1].real(), h[i + 1].imag()));
  };
  B.n = n;
  B.lam.assign(n, zc(0));
  B.W.assign((size_t)n * n, zc(0));
  if (n < 1) {
    err = "empty pencil";
    return false;
  }
  bool real = true, uniform = true;
  for (int t = 0; t <= n; ++t) {
    if (h[t].imag() != 0) real = false;
    if (h[t] != h[0]) uniform = false;
  }
  if (mass)
    for (int t = 0; t < n; ++t) {
      if ((*mass)[t].imag() != 0) real = false;
      if ((*mass)[t] != h[0]) uniform = false;
    }
  std::vector<long double> ord_re(n), ord_im(n);
  std::vector<lc> lamL(n), WL((size_t)n * n);  // WL row-major W[p*n + l]
  if (real && uniform) {
    B.kind = 0;
    const long double hs = h[0].real();
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double sc = std::sqrt(2.0L / (hs * (n + 1)));
    // natural mode order: column c holds sine mode l = c + 1, so that the forward and
    // inverse transforms of a U block are plain DST-I (the fast sine-transform kernel)
    for (int c = 0; c < n; ++c) {
      int l = c + 1;
      long double sl = std::sin(pi * l / (2.0L * (n + 1)));
      lamL[c] = lc(-(4.0L / (hs * hs)) * sl * sl, 0);
      for (int p = 0; p < n; ++p) WL[(size_t)p * n + c] = lc(sc * std::sin(pi * (long double)(p + 1) * l / (n + 1)), 0);
    }
  } else {
    B.kind = real ? 1 : 2;
    // pencil entries in long double
    std::vector<lc> hh(n), s(n), d(n), e(n > 1 ? n - 1 : 0);
    for (int i = 0; i < n; ++i) {
      lc h0(h[i].real(), h[i].imag()), h1(h[i + 1].real(), h[i + 1].imag());
      hh[i] = hhat(i);
      s[i] = lc(1) / std::sqrt(hh[i]);
      d[i] = -(lc(1) / h0 + lc(1) / h1) * s[i] * s[i];
    }
    for (int i = 0; i + 1 < n; ++i) {
      lc h1(h[i + 1].real(), h[i + 1].imag());
      e[i] = (lc(1) / h1) * s[i] * s[i + 1];
    }
    bool palin = n >= 2;
    for (int t = 0; t <= n && palin; ++t) palin = (h[t] == h[n - t]);
    for (int t = 0; mass && t < n && palin; ++t) palin = ((*mass)[t] == (*mass)[n - 1 - t]);
    std::vector<lc> lamv;
    std::vector<lc> V;  // column-major n x n
    if (!palin) {
      if (!tridiag_eig(d, e, lamv, V)) {
        err = "QL iteration failed";
        return false;
      }
    } else {
      const int k = n / 2;
      const long double r2 = std::sqrt(2.0L);
      std::vector<lc> de, ee, dod, eod, le, lo, Ve, Vo;
      if (n % 2 == 0) {
        de.assign(d.begin(), d.begin() + k);
        dod = de;
        de[k - 1] += e[k - 1];
        dod[k - 1] -= e[k - 1];
        ee.assign(e.begin(), e.begin() + (k - 1));
        eod = ee;
      } else {
        de.assign(d.begin(), d.begin() + k + 1);
        ee.assign(e.begin(), e.begin() + k);
        ee[k - 1] = r2 * e[k - 1];
        dod.assign(d.begin(), d.begin() + k);
        eod.assign(e.begin(), e.begin() + (k > 0 ? k - 1 : 0));
      }
      if (!tridiag_eig(de, ee, le, Ve)) {
        err = "QL iteration failed (even half)";
        return false;
      }
      if (!dod.empty() && !tridiag_eig(dod, eod, lo, Vo)) {
        err = "QL iteration failed (odd half)";
        return false;
      }
      const int ne = (int)le.size(), no = (int)lo.size();
      lamv.resize(n);
      V.assign((size_t)n * n, lc(0));
      for (int j = 0; j < ne; ++j) {
        lamv[j] = le[j];
        for (int i = 0; i < k; ++i) {
          lc y = Ve[i + (size_t)ne * j];
          V[i + (size_t)n * j] = y / r2;
          V[(n - 1 - i) + (size_t)n * j] = y / r2;
        }
        if (n % 2 == 1) V[k + (size_t)n * j] = Ve[k + (size_t)ne * j];  // sqrt2 * gamma / sqrt2
      }
      for (int j = 0; j < no; ++j) {
        lamv[ne + j] = lo[j];
        for (int i = 0; i < k; ++i) {
          lc y = Vo[i + (size_t)no * j];
          V[i + (size_t)n * (ne + j)] = y / r2;
          V[(n - 1 - i) + (size_t)n * (ne + j)] = -y / r2;
        }
      }
    }
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
      return lamv[a].real() < lamv[b].real() || (lamv[a].real() == lamv[b].real() && lamv[a].imag() < lamv[b].imag());
    });
    for (int c = 0; c < n; ++c) {
      int j = idx[c];
      lamL[c] = lamv[j];
      for (int p = 0; p < n; ++p) WL[(size_t)p * n + c] = s[p] * V[p + (size_t)n * j];
    }
  }
  for (int c = 0; c < n; ++c) B.lam[c] = zc((double)lamL[c].real(), (double)lamL[c].imag());
  for (size_t q = 0; q < (size_t)n * n; ++q) B.W[q] = zc((double)WL[q].real(), (double)WL[q].imag());
  // diagnostics (long double): pencil residual (all columns), biorthonormality (sampled)
  {
    long double anorm = 0, wmax = 0, res = 0;
    std::vector<lc> hh(n), a_sub(n), a_dia(n), a_sup(n);
    for (int i = 0; i < n; ++i) {
      lc h0(h[i].real(), h[i].imag()), h1(h[i + 1].real(), h[i + 1].imag());
      hh[i] = hhat(i);
      a_sub[i] = i > 0 ? lc(1) / h0 : lc(0);
      a_sup[i] = i + 1 < n ? lc(1) / h1 : lc(0);
      a_dia[i] = -(lc(1) / h0 + lc(1) / h1);
      anorm = std::max(anorm, std::abs(a_sub[i]) + std::abs(a_dia[i]) + std::abs(a_sup[i]));
    }
    for (size_t q = 0; q < (size_t)n * n; ++q) wmax = std::max(wmax, (long double)std::abs(B.W[q]));
    for (int c = 0; c < n; ++c) {
      lc lm(B.lam[c].real(), B.lam[c].imag());
      for (int p = 0; p < n; ++p) {
        auto w = [&](int pp) { return lc(B.W[(size_t)pp * n + c].real(), B.W[(size_t)pp * n + c].imag()); };
        lc aw = a_dia[p] * w(p);
        if (p > 0) aw += a_sub[p] * w(p - 1);
        if (p + 1 < n) aw += a_sup[p] * w(p + 1);
        res = std::max(res, std::abs(aw - hh[p] * w(p) * lm));
      }
    }
    B.residual = (double)(res / (anorm * (wmax > 0 ? wmax : 1)));
    long double bio = 0;
    const int step = n > 48 ? n / 24 : 1;
    for (int c1 = 0; c1 < n; c1 += step) {
      for (int c2 = 0; c2 < n; ++c2) {
        lc acc = 0;
        for (int p = 0; p < n; ++p)
          acc += lc(B.W[(size_t)p * n + c1].real(), B.W[(size_t)p * n + c1].imag()) * hh[p] *
                 lc(B.W[(size_t)p * n + c2].real(), B.W[(size_t)p * n + c2].imag());
        if (c1 == c2) acc -= 1;
        bio = std::max(bio, std::abs(acc));
      }
    }
    B.biorth = (double)bio;
  }
  return true;
}


// ---------------------------------------------------------------------------------------
// z-direction modal basis for step 5 (build design): the global z-systems of
// PAPER.md:56 are T(s) = A' + s E with A' = tridiag(a, g, c) real symmetric (a_k = c_{k-1})
// and E = diag(e) > 0 (e_k = sigma_k hz^_k, reading R1).  With A' Z = E Z Theta and
// Z^T E Z = I, T(s)^{-1} = Z (Theta + s)^{-1} Z^T.  S = E^{-1/2} A' E^{-1/2} is real symmetric
// tridiagonal; its eigenpairs come from the implicit QL iteration with Wilkinson shifts and
// accumulated plane rotations (orthogonal to working precision), in long double.
static bool ql_real_vectors(std::vector<long double>& d, std::vector<long double> e, std::vector<long double>& V) {
  const int n = (int)d.size();
  e.resize(n, 0.0L);  // e[i] couples i and i+1; e[n-1] = 0
  V.assign((size_t)n * n, 0.0L);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0L;  // V[row * n + col]
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const long double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= LDBL_EPSILON * dd) break;
      }
      if (m == l) break;
      if (++iter > 80) return false;
      // shift from the leading 2x2 block (eigenvalue closer to d[l])
      long double g = (d[l + 1] - d[l]) / (2.0L * e[l]);
      long double r = std::hypot(g, 1.0L);
      g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      long double s = 1.0L, c = 1.0L, p = 0.0L;
      int i;
      bool deflated = false;
      for (i = m - 1; i >= l; --i) {
        long double f = s * e[i];
        const long double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0L) {  // underflow: split the matrix here
          d[i + 1] -= p;
          e[m] = 0.0L;
          deflated = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0L * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        for (int k = 0; k < n; ++k) {  // accumulate the rotation on columns i, i+1
          f = V[(size_t)k * n + i + 1];
          V[(size_t)k * n + i + 1] = s * V[(size_t)k * n + i] + c * f;
          V[(size_t)k * n + i] = c * V[(size_t)k * n + i] - s * f;
        }
      }
      if (deflated) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0L;
    } while (m != l);
  }
  return true;
}

bool z_modal_basis(const std::vector<double>& a, const std::vector<double>& g, const std::vector<double>& c,
                   const std::vector<double>& e, std::vector<double>& theta, std::vector<double>& Z,
                   double& residual, double& orth, std::string& err) {
  const int n = (int)g.size();
  if (n < 1) { err = "empty z pencil"; return false; }
  std::vector<long double> sq(n), d(n), off(n > 1 ? n - 1 : 0), V;
  for (int k = 0; k < n; ++k) {
    if (!(e[k] > 0)) { err = "z mass not positive"; return false; }
    sq[k] = std::sqrt((long double)e[k]);
    d[k] = (long double)g[k] / (long double)e[k];
  }
  for (int k = 0; k + 1 < n; ++k) {
    if (c[k] != a[k + 1]) { err = "z operator not symmetric"; return false; }
    off[k] = (long double)c[k] / (sq[k] * sq[k + 1]);
  }
  if (!ql_real_vectors(d, off, V)) { err = "QL iteration did not converge (z pencil)"; return false; }
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int p, int q) { return d[p] < d[q]; });
  theta.assign(n, 0.0);
  Z.assign((size_t)n * n, 0.0);  // Z[k * n + t]
  std::vector<long double> ZL((size_t)n * n);
  for (int t = 0; t < n; ++t) {
    theta[t] = (double)d[idx[t]];
    for (int k = 0; k < n; ++k) {
      ZL[(size_t)k * n + t] = V[(size_t)k * n + idx[t]] / sq[k];
      Z[(size_t)k * n + t] = (double)ZL[(size_t)k * n + t];
    }
  }
  // diagnostics on the rounded (double) basis: pencil residual and E-orthonormality
  long double anorm = 0, res = 0, orr = 0, zmax = 0;
  for (int k = 0; k < n; ++k)
    anorm = std::max(anorm, std::fabs((long double)a[k]) + std::fabs((long double)g[k]) + std::fabs((long double)c[k]));
  for (auto v : Z) zmax = std::max(zmax, std::fabs((long double)v));
  for (int t = 0; t < n; ++t)
    for (int k = 0; k < n; ++k) {
      long double az = (long double)g[k] * Z[(size_t)k * n + t];
      if (k > 0) az += (long double)a[k] * Z[(size_t)(k - 1) * n + t];
      if (k + 1 < n) az += (long double)c[k] * Z[(size_t)(k + 1) * n + t];
      res = std::max(res, std::fabs(az - (long double)theta[t] * e[k] * Z[(size_t)k * n + t]));
    }
  for (int t1 = 0; t1 < n; ++t1)
    for (int t2 = t1; t2 < n; ++t2) {
      long double acc = 0;
      for (int k = 0; k < n; ++k) acc += (long double)Z[(size_t)k * n + t1] * e[k] * Z[(size_t)k * n + t2];
      if (t1 == t2) acc -= 1;
      orr = std::max(orr, std::fabs(acc));
    }
  residual = (double)(res / (anorm * (zmax > 0 ? zmax : 1)));
  orth = (double)orr;
  return true;
}

// Eigenvalues theta_t of the z pencil A' z = theta E z (complex tables allowed: complex sigma or
// lambda, reading R11): the complex-symmetric tridiagonal S = E^{-1/2} A' E^{-1/2} (principal
// square roots) by implicit QL in long double.  Used for the resonance margins
// min |lambda_l + mu_m + theta_t| of the block and global z-systems T_lm = A' + (lambda_l + mu_m) E.
bool z_pencil_values(const std::vector<zc>& a, const std::vector<zc>& g, const std::vector<zc>& c,
                     const std::vector<zc>& e, std::vector<zc>& theta, std::string& err) {
  const int n = (int)g.size();
  if (n < 1) { err = "empty z pencil"; return false; }
  std::vector<lc> sq(n), d(n), off(n > 1 ? n - 1 : 0);
  for (int k = 0; k < n; ++k) {
    if (e[k] == zc(0)) { err = "z mass has a zero entry"; return false; }
    sq[k] = std::sqrt(lc(e[k]));
    d[k] = lc(g[k]) / lc(e[k]);
  }
  for (int k = 0; k + 1 < n; ++k) {
    if (c[k] != a[k + 1]) { err = "z operator not symmetric"; return false; }
    off[k] = lc(c[k]) / (sq[k] * sq[k + 1]);
  }
  if (!ql_values(d, off)) { err = "QL iteration did not converge (z pencil values)"; return false; }
  theta.resize(n);
  for (int t = 0; t < n; ++t) theta[t] = zc((double)d[t].real(), (double)d[t].imag());
  return true;
}

}  // namespace lfds
