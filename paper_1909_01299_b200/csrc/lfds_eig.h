// Host 1D generalized eigensolver; see lfds_eig.cpp.
#pragma once
#include <complex>
#include <string>
#include <vector>

namespace lfds {

using zc = std::complex<double>;

struct Basis {
  int n = 0;
  int kind = 0;              // 0 = U (uniform real steps, exact sine modes), 1 = R (real), 2 = C (complex)
  std::vector<zc> lam;       // n eigenvalues: ascending (Re, Im) for R/C, natural sine order l = 1..n for U (R14)
  std::vector<zc> W;         // row-major W[p*n + l]; A W = M W diag(lam), W^T M W = I
  double residual = 0;       // max_l ||A w_l - lam_l M w_l||_inf / (||A||_inf max|W|)
  double biorth = 0;         // max |W^T M W - I| over sampled columns
};

// Eigenbasis of the Dirichlet pencil of the N+1 steps h (N interior nodes).  mass (N values)
// replaces the control volumes (h_{i-1} + h_i)/2 as the diagonal of M when given (the
// Lebedev-grid primary pencil of the Maxwell solve, lfds_mw.cpp).
bool pencil_basis(const std::vector<zc>& h, Basis& B, std::string& err, const std::vector<zc>* mass = nullptr);

// z modal basis for step 5 (real z tables only): A' Z = E Z diag(theta), Z^T E Z = I, with
// A' = tridiag(a, g, c) (a[k] couples k-1, c[k] couples k+1; a[k+1] == c[k]) and E = diag(e).
// Z is row-major Z[k * n + t]; theta ascending.  residual = max |A'z - theta E z| /
// (||A'||_inf max|Z|), orth = max |Z^T E Z - I|.
bool z_modal_basis(const std::vector<double>& a, const std::vector<double>& g, const std::vector<double>& c,
                   const std::vector<double>& e, std::vector<double>& theta, std::vector<double>& Z,
                   double& residual, double& orth, std::string& err);

// Eigenvalues of the (possibly complex) z pencil A' z = theta E z, same table convention.
bool z_pencil_values(const std::vector<zc>& a, const std::vector<zc>& g, const std::vector<zc>& c,
                     const std::vector<zc>& e, std::vector<zc>& theta, std::string& err);

}  // namespace lfds
