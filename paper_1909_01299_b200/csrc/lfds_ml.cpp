// Multi-level (nested) variant of the blocked separable solve — PAPER.md:77-79 (remark): "by
// employing multiple mutually embedded partitions of S" the N^{3/2} cost of the interface step
// drops towards N log N per direction, at the price of "multiple (on each level of embedding)
// solution of block-tridiagonal systems".  SURVEY §8(f) NEXT #4.
//
// Three levels: the grid S, coarse blocks C (interfaces I_c), and fine blocks inside every coarse
// block (interfaces I_f, a superset of I_c).  The two-level method of PAPER.md:63-73 runs on the
// coarse partition, with every coarse-block problem (steps 2 and 6 of the coarse level: a
// Dirichlet problem on C) solved by the two-level method of that block's own fine partition,
// whose interface step uses C's bases (size n_C) instead of the global ones (size N):
//   1. v_C = A_C^{-1} M f_C on every coarse block (homogeneous Dirichlet on dC):  fine two-level
//      solve of the sub-grid C (its own lfds_plan);  u = v, zero on the coarse planes;
//   2. r_b = M f - A u on the coarse planes (lfds_residual, gathered into RX / RY);
//   3. w on the coarse planes from the global bases (the coarse plan's step 5: lfds_solve_phase 2,
//      then the plane inverse and u = w on the planes: phase 6);
//   4. u_C = A_C^{-1} (M f_C - A_{C,dC} w) on every coarse block (the Dirichlet lifting of reading
//      R8 folded into the right side: f_C - sigma_k w / (h hx^) on the rows next to the coarse
//      faces), again by the fine two-level solve of C.
// Exact, like the two-level method: u = A^{-1} M f up to rounding.  The coarse plan's own block
// transforms are never used.
#include <cuda_runtime.h>

#include <algorithm>
#include <complex>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lfds.h"
#include "lfds_internal.h"

using lfds::MlLift;
using lfds::PlaneLayout;
using zc = std::complex<double>;

namespace {
thread_local std::string g_ml_err;
int mlfail(int code, const char* msg) {
  g_ml_err = msg;
  return code;
}
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

struct lfds_ml {
  lfds_plan* coarse = nullptr;
  struct Sub {
    lfds_plan* plan = nullptr;
    int x0 = 0, nxc = 0, y0 = 0, nyc = 0;  // 0-based first node and sizes of the coarse block
    int aL = -1, aR = -1, bB = -1, bT = -1;  // coarse plane of each face (-1: outer boundary)
    double2 cL{}, cR{}, cB{}, cT{};          // 1 / (h hx^) of each face coupling
  };
  std::vector<Sub> sub;
  int nx = 0, ny = 0, nz = 0, ncx = 0, ncy = 0;
  int* d_ifx = nullptr;
  int* d_ify = nullptr;
  double2* d_sig = nullptr;
  size_t ws_coarse = 0, ws_sub = 0, vol_sub = 0;
  PlaneLayout lay{};
};

extern "C" {

const char* lfds_ml_last_error(void) { return g_ml_err.c_str(); }

void lfds_ml_destroy(lfds_ml* M) {
  if (!M) return;
  if (M->coarse) lfds_destroy(M->coarse);
  for (auto& s : M->sub)
    if (s.plan) lfds_destroy(s.plan);
  cudaFree(M->d_ifx);
  cudaFree(M->d_ify);
  cudaFree(M->d_sig);
  delete M;
}

int lfds_ml_setup(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                  const lfds_z* sigma_node, const lfds_z* sigma_edge, lfds_z lambda, int n_cx, const int* cx, int n_cy,
                  const int* cy, int n_fx, const int* fx, int n_fy, const int* fy, const lfds_options* opt,
                  lfds_ml** out) {
  if (!out) return mlfail(LFDS_EINVAL, "out is NULL");
  *out = nullptr;
  lfds_options o;
  if (opt) o = *opt;
  else lfds_default_options(&o);
  if (o.dtype != LFDS_C128 || o.device < 0) return mlfail(LFDS_EINVAL, "lfds_ml: complex128 device plans only");
  if (o.refine != 0) return mlfail(LFDS_EINVAL, "lfds_ml: no refinement");
  o.profile = 0;
  // every coarse interface must be a fine one
  for (int a = 0; a < n_cx; ++a)
    if (std::find(fx, fx + n_fx, cx[a]) == fx + n_fx) return mlfail(LFDS_EINVAL, "coarse x interface not in the fine set");
  for (int b = 0; b < n_cy; ++b)
    if (std::find(fy, fy + n_fy, cy[b]) == fy + n_fy) return mlfail(LFDS_EINVAL, "coarse y interface not in the fine set");
  std::unique_ptr<lfds_ml> M(new lfds_ml());
  M->nx = nx; M->ny = ny; M->nz = nz; M->ncx = n_cx; M->ncy = n_cy;
  int rc;
  {  // the coarse plan: its step 5 (global bases over the coarse planes) and residual only
    lfds_options oc = o;
    oc.graph = 0;
    if ((rc = lfds_setup_grid(nx, hx, ny, hy, nz, hz, sigma_node, sigma_edge, lambda, n_cx, cx, n_cy, cy, &oc,
                              &M->coarse))) {
      g_ml_err = std::string("coarse plan: ") + lfds_last_error();
      return rc;
    }
  }
  // coarse blocks and their fine partitions (sub-grids of steps h_{X0-1} .. h_{X1})
  std::vector<int> xc = {0}, yc = {0};
  xc.insert(xc.end(), cx, cx + n_cx); xc.push_back(nx + 1);
  yc.insert(yc.end(), cy, cy + n_cy); yc.push_back(ny + 1);
  auto hh = [](const lfds_z* h, int node) {  // control volume of 1-based node
    return 0.5 * (zc(h[node - 1].re, h[node - 1].im) + zc(h[node].re, h[node].im));
  };
  for (int j = 0; j + 1 < (int)yc.size(); ++j)
    for (int i = 0; i + 1 < (int)xc.size(); ++i) {
      lfds_ml::Sub S;
      const int X0 = xc[i] + 1, X1 = xc[i + 1] - 1, Y0 = yc[j] + 1, Y1 = yc[j + 1] - 1;
      S.x0 = X0 - 1; S.nxc = X1 - X0 + 1; S.y0 = Y0 - 1; S.nyc = Y1 - Y0 + 1;
      std::vector<int> fxs, fys;
      for (int a = 0; a < n_fx; ++a)
        if (fx[a] > X0 && fx[a] < X1) fxs.push_back(fx[a] - X0 + 1);
      for (int b = 0; b < n_fy; ++b)
        if (fy[b] > Y0 && fy[b] < Y1) fys.push_back(fy[b] - Y0 + 1);
      lfds_options os = o;
      os.graph = 1;  // constant buffers per sub-plan: its launches replay as a CUDA graph
      if ((rc = lfds_setup_grid(S.nxc, hx + (X0 - 1), S.nyc, hy + (Y0 - 1), nz, hz, sigma_node, sigma_edge, lambda,
                                (int)fxs.size(), fxs.data(), (int)fys.size(), fys.data(), &os, &S.plan))) {
        g_ml_err = std::string("coarse block plan: ") + lfds_last_error();
        M->sub.push_back(S);
        lfds_ml_destroy(M.release());
        return rc;
      }
      auto cpl = [&](const lfds_z* h, int step, int node) {
        const zc c = 1.0 / (zc(h[step].re, h[step].im) * hh(h, node));
        return make_double2(c.real(), c.imag());
      };
      if (i > 0) { S.aL = i - 1; S.cL = cpl(hx, X0 - 1, X0); }
      if (i + 1 < (int)xc.size() - 1) { S.aR = i; S.cR = cpl(hx, X1, X1); }
      if (j > 0) { S.bB = j - 1; S.cB = cpl(hy, Y0 - 1, Y0); }
      if (j + 1 < (int)yc.size() - 1) { S.bT = j; S.cT = cpl(hy, Y1, Y1); }
      M->sub.push_back(S);
      M->ws_sub = std::max(M->ws_sub, lfds_workspace_bytes(S.plan, 1));
      M->vol_sub = std::max(M->vol_sub, (size_t)S.nxc * S.nyc * nz * 16);
    }
  M->ws_coarse = lfds_workspace_bytes(M->coarse, 1);
  if (!M->ws_coarse || !M->ws_sub) {
    lfds_ml_destroy(M.release());
    return mlfail(LFDS_ECUDA, "workspace query failed");
  }
  if ((rc = lfds::plane_layout(M->coarse, &M->lay))) {
    lfds_ml_destroy(M.release());
    return mlfail(rc, "coarse plane layout");
  }
  std::vector<double2> sig(nz);
  for (int k = 0; k < nz; ++k) sig[k] = make_double2(sigma_node[k].re, sigma_node[k].im);
  cudaError_t e = cudaMalloc(&M->d_ifx, sizeof(int) * std::max(1, n_cx));
  if (e == cudaSuccess) e = cudaMalloc(&M->d_ify, sizeof(int) * std::max(1, n_cy));
  if (e == cudaSuccess) e = cudaMalloc(&M->d_sig, sizeof(double2) * nz);
  if (e == cudaSuccess && n_cx) e = cudaMemcpy(M->d_ifx, cx, sizeof(int) * n_cx, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n_cy) e = cudaMemcpy(M->d_ify, cy, sizeof(int) * n_cy, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(M->d_sig, sig.data(), sizeof(double2) * nz, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    lfds_ml_destroy(M.release());
    return mlfail(LFDS_ECUDA, cudaGetErrorString(e));
  }
  *out = M.release();
  return LFDS_OK;
}

size_t lfds_ml_workspace_bytes(const lfds_ml* M) {
  if (!M) return 0;
  const size_t vol = (size_t)M->nx * M->ny * M->nz * 16;
  return al256(M->ws_coarse) + al256(M->ws_sub) + 2 * al256(M->vol_sub) + al256(vol);
}

// copy a coarse block between the full field [nz][ny][nx] and a packed [nz][nyc][nxc] array
static cudaError_t block_copy(const lfds_ml::Sub& S, int nx, int ny, int nz, void* full, void* packed, bool to_packed,
                              cudaStream_t st) {
  cudaMemcpy3DParms p{};
  p.extent = make_cudaExtent((size_t)S.nxc * 16, S.nyc, nz);
  p.kind = cudaMemcpyDeviceToDevice;
  cudaPitchedPtr F = make_cudaPitchedPtr(full, (size_t)nx * 16, (size_t)nx * 16, ny);
  cudaPitchedPtr B = make_cudaPitchedPtr(packed, (size_t)S.nxc * 16, (size_t)S.nxc * 16, S.nyc);
  if (to_packed) {
    p.srcPtr = F; p.srcPos = make_cudaPos((size_t)S.x0 * 16, S.y0, 0);
    p.dstPtr = B; p.dstPos = make_cudaPos(0, 0, 0);
  } else {
    p.srcPtr = B; p.srcPos = make_cudaPos(0, 0, 0);
    p.dstPtr = F; p.dstPos = make_cudaPos((size_t)S.x0 * 16, S.y0, 0);
  }
  return cudaMemcpy3DAsync(&p, st);
}

int lfds_ml_solve(lfds_ml* M, const void* f_dev, void* u_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!M || !f_dev || !u_dev || !ws) return mlfail(LFDS_EINVAL, "bad arguments");
  if (ws_bytes < lfds_ml_workspace_bytes(M)) return mlfail(LFDS_EINVAL, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  void* wsc = w;
  void* wss = w + al256(M->ws_coarse);
  char* fC = w + al256(M->ws_coarse) + al256(M->ws_sub);
  char* uC = fC + al256(M->vol_sub);
  lfds_z* r = reinterpret_cast<lfds_z*>(uC + al256(M->vol_sub));
  const size_t vol = (size_t)M->nx * M->ny * M->nz * 16;
  int rc;
  cudaError_t e;
  auto cuda = [&](cudaError_t x) { return x == cudaSuccess ? LFDS_OK : mlfail(LFDS_ECUDA, cudaGetErrorString(x)); };
  auto sub_solve = [&](const lfds_ml::Sub& S) -> int {
    const int q = lfds_solve(S.plan, fC, uC, 1, wss, M->ws_sub, st);
    if (q) g_ml_err = std::string("coarse block solve: ") + lfds_last_error();
    return q;
  };
  // 1. v on every coarse block (homogeneous Dirichlet on its faces); u = v, 0 on the coarse planes
  if ((rc = cuda(cudaMemsetAsync(u_dev, 0, vol, st)))) return rc;
  for (auto& S : M->sub) {
    if ((rc = cuda(block_copy(S, M->nx, M->ny, M->nz, const_cast<void*>(f_dev), fC, true, st)))) return rc;
    if ((rc = sub_solve(S))) return rc;
    if ((rc = cuda(block_copy(S, M->nx, M->ny, M->nz, u_dev, uC, false, st)))) return rc;
  }
  // 2. r_b = M f - A u on the coarse planes (v = 0 there), into the coarse plan's RX / RY
  if ((rc = lfds_residual(M->coarse, u_dev, f_dev, r, 1, 0, nullptr, stream))) {
    g_ml_err = std::string("coarse residual: ") + lfds_last_error();
    return rc;
  }
  double2* IF = reinterpret_cast<double2*>(static_cast<char*>(wsc) + M->lay.off_if);
  if ((e = lfds::launch_ml_gather(reinterpret_cast<const double2*>(r), M->nx, M->ny, M->nz, M->d_ifx, M->ncx,
                                  M->d_ify, M->ncy, IF + M->lay.rx, IF + M->lay.ry, st)))
    return cuda(e);
  // 3. w on the coarse planes (global bases), u = w there
  for (int ph : {2, 6})
    if ((rc = lfds_solve_phase(M->coarse, ph, f_dev, u_dev, 1, wsc, M->ws_coarse, stream))) {
      g_ml_err = std::string("coarse step 5: ") + lfds_last_error();
      return rc;
    }
  // 4. every coarse block again, with the lifting of w on its faces folded into the right side
  for (auto& S : M->sub) {
    if ((rc = cuda(block_copy(S, M->nx, M->ny, M->nz, const_cast<void*>(f_dev), fC, true, st)))) return rc;
    MlLift L{};
    L.nxc = S.nxc; L.nyc = S.nyc; L.nz = M->nz;
    L.cL = S.cL; L.cR = S.cR; L.cB = S.cB; L.cT = S.cT;
    L.ldx = M->ny; L.ldy = M->nx; L.ox = S.y0; L.oy = S.x0;
    const double2* WX = IF + M->lay.wx;
    const double2* WY = IF + M->lay.wy;
    const int64_t px = (int64_t)M->nz * M->ny, py = (int64_t)M->nz * M->nx;
    L.wL = S.aL >= 0 ? WX + S.aL * px : nullptr;
    L.wR = S.aR >= 0 ? WX + S.aR * px : nullptr;
    L.wB = S.bB >= 0 ? WY + S.bB * py : nullptr;
    L.wT = S.bT >= 0 ? WY + S.bT * py : nullptr;
    if ((e = lfds::launch_ml_lift(L, M->d_sig, reinterpret_cast<const double2*>(fC), reinterpret_cast<double2*>(fC),
                                  st)))
      return cuda(e);
    if ((rc = sub_solve(S))) return rc;
    if ((rc = cuda(block_copy(S, M->nx, M->ny, M->nz, u_dev, uC, false, st)))) return rc;
  }
  return LFDS_OK;
}

int lfds_ml_get_plans(const lfds_ml* M, int* n_sub) {
  if (!M || !n_sub) return LFDS_EINVAL;
  *n_sub = (int)M->sub.size();
  return LFDS_OK;
}

}  // extern "C"
