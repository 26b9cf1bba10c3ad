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

// Eigenbasis of the Dirichlet pencil of the N+1 steps h (N interior nodes).
bool pencil_basis(const std::vector<zc>& h, Basis& B, std::string& err);

}  // namespace lfds
