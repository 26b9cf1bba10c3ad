// Internal declarations shared by the host orchestration (lfds_host.cpp) and the
// sm_100a kernels (lfds_kernels.cu).  Not part of the public ABI (include/lfds.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace lfds {

// Device buffers addressed by descriptors (offsets are in elements of the buffer's type:
// complex128 everywhere except B_F / B_U of an LFDS_F64 plan, which are float64).
enum BufId { B_TAB = 0, B_F = 1, B_U = 2, B_MS = 3, B_T1 = 4, B_IF = 5, B_RED = 6, B_CK = 7, NBUF = 8 };

struct Bufs {
  void* p[NBUF];
};

// Strided batched complex GEMM  C(i, n) (+)= sum_j A(i, j) * B(j, n),  n = (n1, n2).
//   A(i,j) = TAB[a_off + i*sAi + j*sAj]            (always complex, in the plan tables)
//   B(j,n) = buf[b_buf][b_off + j*sBj + n1*sB1 + n2*sB2]
//   C(i,n) = buf[c_buf][c_off + i*sCi + n1*sC1 + n2*sC2]
// All four transform passes of a block, the sparse global transforms
// of step 5, the interface-adjacent evaluations of step 3 and the
// face transforms of step 6 are instances of this one contraction.
enum GemmFlags { G_BREAL = 1, G_CREAL = 2, G_ACCUM = 4 };
struct GemmDesc {
  int64_t a_off, sAi, sAj;
  int64_t b_off, sBj, sB1, sB2;
  int64_t c_off, sCi, sC1, sC2;
  int M, K, N1, N2;
  int b_buf, c_buf, flags, pad;
  double scale;                // used by the sine-transform kernel (alpha)
};

// z-tables: per row k the tridiagonal row (a_k x_{k-1} + (g_k + s e_k) x_k + c_k x_{k+1})
// of T(s) = A_z + lambda M_z + s M_z^sigma (reading R1); 'row-scaled' tables are divided
// by hz^_k so that the RHS of a block z-solve is the f-unit transform (no M_z factor).
struct ZTab {
  int64_t a, g, c, e;  // offsets in TAB (nz complex each)
};

// One block for the block-pass z-solves.
struct ZBlock {
  int64_t ms_off;              // offset of this block's mode space [r][k][m][l] in B_MS (and T1)
  int nx, ny;                  // interior sizes (modes)
  int buf, pad_;               // mode-space buffer (B_MS, or B_T1 for step 5); pad_ = 1: real eigenvalues
  int64_t lamx, lamy;          // eigenvalue offsets in TAB
  // pass-2 lifting (reading R8): l~[l,m,k] = -sigma_k (cL Wx[0,l] GL[m,k] + cR Wx[n-1,l] GR[m,k]
  //                                               + cB Wy[0,m] GB[l,k] + cT Wy[n-1,m] GT[l,k])
  int64_t wx0, wx1, wy0, wy1;  // offsets in TAB of W rows (first / last interior node)
  int64_t gL, gR, gB, gT;      // offsets in B_IF of the face transforms, [r*nz + k][m or l]; -1 = none
  int64_t fstride;             // row stride of the face-transform arrays
  double2 cL, cR, cB, cT;      // coupling coefficients 1/h across each face (0 at outer boundary)
};

// Step-5 global sweep parameters (Eq. (fdmtrprjfrerr)).
struct GSweep {
  int nx, ny, nifx, nify, nz, R;
  int64_t lamx, lamy;          // global eigenvalues (TAB)
  int64_t wxi, wyi;            // W_x[I_a, l] (nifx x nx), W_y[I_b, m] (nify x ny)  (TAB)
  int64_t r1, r2;              // R1[a][r][k][m], R2[b][r][k][l]  (B_IF)
  int64_t what;                // W^[r][k][m][l] output (B_T1)
  int l_begin, l_end;          // global x-modes swept by this rank (block sharding); all: 0, nx
};

// Interface residual (step 4).
struct IfaceRes {
  int nx, ny, nz, R, nifx, nify, dtype;
  int64_t ifx, ify;            // int arrays (device) of 1-based interface nodes
  int64_t hx, hy, hhx, hhy, hhz, sig;   // TAB offsets (steps, control volumes, sigma_k)
  int64_t rx, ry;              // out: RX[a][r][k][q] (all q), RY[b][r][k][p] (0 at p in I_x) (B_IF)
  int64_t vxo, vyo;            // in: v next to the faces, VX[blk][e][r][k][qpad], VY[blk][e][r][k][ppad]
  int64_t blk_of_x, blk_of_y;  // int arrays: block index along the axis for each node (or -1)
  int64_t xlo, ylo;            // int arrays: first node of each block along the axis
  int nbx, nby;
  int qpad, ppad;              // padded row lengths of the step-3 arrays VX / VY
  const int* own;              // per block: 1 if this rank computed its v (block sharding)
  int with_b;                  // 1: add the b = M f term (exactly one rank does)
};

// Two-sided projection of mode planes (lfds_proj.cu): G[e][p][m] = sum_l Wr[e][l] X[p][m][l],
// H[e][p][l] = sum_m Wc[e][m] X[p][m][l] (step 3 edge values, E1 = E2 = 2).
struct PDesc {
  int64_t x_off, ps;           // plane p of X at x_off + p*ps in buffer x_buf; row m at + m*nx
  int x_buf, nx, ny, nplanes;
  int E1, E2, pad0, pad1;
  int64_t wr, wr_es;           // TAB: Wr[e][l] at wr + e*wr_es + l
  int64_t wc, wc_es;           // TAB: Wc[e][m] at wc + e*wc_es + m
  int64_t g_off, g_es, g_ps;   // IF: G[e][p][m] at g_off + e*g_es + p*g_ps + m
  int64_t h_off, h_es, h_ps;   // IF: H[e][p][l] at h_off + e*h_es + p*h_ps + l
};
cudaError_t launch_proj(const PDesc* d_descs, int ndesc, int max_nx, int maxE, int maxplanes, cudaStream_t st,
                        const Bufs& bufs);

// Step-5 projections of the global correction (lfds_proj.cu, DMMA): P1 = W_x[I,:] w^ (over l),
// P2 = W_y[I,:] w^ (over m), one read of w^[p][m][l] (plane stride nx*ny).  P1 partials per
// l-chunk of 256 columns at g_off + lc*g_lcs + e*g_es + p*g_ps + m, summed into p1_off.
struct ProjM {
  int nx, ny, nplanes, E1, E2, nlc, x_buf, pad;
  int l_begin, l_end;          // columns l in [l_begin, l_end) (block sharding: this rank's x-modes)
  int64_t x_off;
  int64_t wr, wc;              // TAB: Wr[e][l] (row stride nx), Wc[e][m] (row stride ny)
  int64_t g_off, g_lcs, g_es, g_ps;
  int64_t p1_off, p1_es;
  int64_t h_off, h_es, h_ps;
};
int projm_chunks(int nx);

// Step 5 in z-modal form (lfds_modal.cu): P1~, P2~ from R1~, R2~ for every z-mode t.
struct S5M {
  int nx, ny, nz, R, nifx, nify;
  int l_begin, l_end;          // this rank's global x-modes
  int nmt;                     // m-tiles (P2 partials)
  int mt_begin, mt_end;        // this rank's m-tiles (y-mode split; all: 0, nmt)
  int64_t lamx, lamy, theta;   // TAB: lambda_l (nx), mu_m (ny), theta_t (nz), complex
  int64_t wxi, wyi;            // TAB: W_x[I_a][l] (nifx x nx), W_y[I_b][m] (nify x ny)
  int64_t r1t, r2t;            // IF: R1~[a][r][t][m], R2~[b][r][t][l]
  int64_t p1t, p2p, p2t;       // IF: P1~[a][r][t][m], P2 partials [b][r][t][mt][l], P2~[b][r][t][l]
};
// Krylov vector kernels (lfds_krylov.cu) for lfds_gmres; dots write partial[blk * 80 + i]
// for blk < KRYLOV_DOT_BLOCKS, i < cnt <= 80
constexpr int KRYLOV_DOT_BLOCKS = 592;
cudaError_t launch_fdie(int64_t n, const double2* v, const double2* dlam, const double2* s, double2* out,
                        cudaStream_t st);
cudaError_t launch_fdie_res(int64_t n, const double2* f, const double2* y, const double2* dlam, const double2* s,
                            double2* out, cudaStream_t st);
cudaError_t launch_dots(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* w, double2* partial,
                        cudaStream_t st, int with_self = 0);
cudaError_t launch_maxpy(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* coef, double2* w,
                         cudaStream_t st);
cudaError_t launch_maxpy_norm(int64_t n, int cnt, const double2* V, int64_t vstride, const double2* coef, double2* w,
                              double2* partial, cudaStream_t st);  // w += V c; partial[blk*80] = ||w||^2 part
cudaError_t launch_scale(int64_t n, double2 alpha, const double2* w, double2* out, cudaStream_t st);

int s5m_ka(int nifx, int nify);   // padded |I| (8 or 16), 0 = unsupported
int s5m_mtiles(int ny);
cudaError_t launch_s5m(const S5M& S, const Bufs& bufs, cudaStream_t st);
cudaError_t launch_projm(const ProjM& P, const Bufs& bufs, cudaStream_t st);

// launchers (lfds_kernels.cu); return cudaGetLastError()
cudaError_t launch_gemm(const GemmDesc* d_descs, int ndesc, int maxM, int maxN, int ldB_hint,
                        const Bufs& bufs, cudaStream_t st);
// persistent form for real bases of at most 32 nodes (maxM, maxK <= 32; k_xsmall)
cudaError_t launch_xform_small(const GemmDesc* d_descs, int ndesc, int maxK, int64_t maxN, bool kcontig,
                               const Bufs& bufs, cudaStream_t st);
cudaError_t launch_xform(const GemmDesc* d_descs, int ndesc, int maxM, int64_t maxN, bool real_s, bool kcontig,
                         const Bufs& bufs, cudaStream_t st);
bool dst_supported(int n);
cudaError_t launch_dst(const GemmDesc* d_descs, int ndesc, int n, int64_t maxN, bool kcontig, const Bufs& bufs,
                       cudaStream_t st);
// Plane (2-D) sine transform of a uniform x uniform block, both axes of length n: per plane
// r < nplanes, C[r][m][l] = ay ax sum_{q,p} S_mq S_lp B[r][q][p] (S = DST-I; rows q/m strided
// by sBr/sCr, p/l contiguous).  One pass over the block instead of an x pass and a y pass.
struct Dst2Desc {
  int64_t b_off, sB1, sBr;
  int64_t c_off, sC1, sCr;
  int64_t tw_off;            // W_L^j table in B_TAB
  int nplanes, b_buf, c_buf, pad;
  double ax, ay;             // DST-I scales of the two axes (dst_fwd or dst_inv)
};
bool dst2_supported(int n);
// Plane (2-D) transform of a block whose x and y bases are both at most 32 nodes long and have no
// sine form (R / C blocks of C5, C3; real or complex matrices per axis): per plane r < nplanes,
//   C[r][m][l] = sum_q Ay[m][q] ( sum_p B[r][q][p] Ax[l][p] )
// (steps 1 and 7 of PAPER.md:66 / :72 in ONE pass over the block: the x-transformed plane stays
// in shared memory).  Ax, Ay: real matrices [out][in] in B_TAB (offsets in doubles), rows q/m
// strided by sBr/sCr, p/l contiguous.
struct XPlaneDesc {
  int64_t b_off, sB1, sBr;
  int64_t c_off, sC1, sCr;
  int64_t ax, ay;
  int nx, ny, nplanes, b_buf, c_buf, pad;
};
// mode: 1 = two-stage ring at 3 CTAs per SM (default), 4 = three-stage ring at 2 CTAs per SM
// cx / cy: the x / y matrices of every descriptor of the launch are complex ([out][in] in B_TAB,
// offsets ax / ay in complex units)
cudaError_t launch_xplane(const XPlaneDesc* d_descs, int ndesc, int nplanes, const Bufs& bufs, cudaStream_t st,
                          int mode = 1, bool cx = false, bool cy = false);
// y (strided) sine passes fed by TMA (k_dstt): one 128-byte tensor map per descriptor, built on
// the host for the descriptor's current input buffer (the map embeds its address)
bool dst_tma_supported(int n);
bool dst_tma_encode(const GemmDesc& D, int n, const Bufs& bufs, void* map_out);
cudaError_t launch_dst_tma(const GemmDesc* d_descs, const void* d_maps, int ndesc, int n, int maxN2, int maxN1,
                           const Bufs& bufs, cudaStream_t st);
cudaError_t launch_dst2(const Dst2Desc* d_descs, int ndesc, int n, int nplanes, const Bufs& bufs, cudaStream_t st);
// z-solves (lfds_zsolve.cu): mode 1 = in place (step 2), 2 = Dirichlet lifting added to v~
// (step 6), 3 = step-5 global modes with the rank-|I| RHS built from R1/R2 (g != NULL)
cudaError_t launch_zsolve(int mode, const ZBlock* d_blocks, int nblocks, int max_nx, int max_ny, int R, int nz,
                          ZTab tab, int64_t sig_off, const GSweep* g, const Bufs& bufs, double* d_minpiv,
                          cudaStream_t st, bool realz);
cudaError_t launch_iface_residual(const IfaceRes& p, const Bufs& bufs, cudaStream_t st);
// wmask (block sharding, else NULL = write all): [a][block row j] then [b][block column i]
// flags of the plane segments this rank writes; intersections only if rank0
cudaError_t launch_write_iface_u(int nx, int ny, int nz, int R, int dtype, int nifx, int nify,
                                 int64_t ifx, int64_t ify, int64_t wx, int64_t wy,
                                 const Bufs& bufs, cudaStream_t st, const int* wmask = nullptr,
                                 int64_t bxo = 0, int64_t byo = 0, int nbx = 1, int nby = 1, int rank0 = 1);
cudaError_t launch_residual(int nx, int ny, int nz, int R, int dtype, int dd, int has_f,
                            int64_t hx, int64_t hy, int64_t hz, int64_t hhx, int64_t hhy, int64_t hhz,
                            int64_t sig, int64_t sige, double2 lam, const int64_t* ddtabs, const void* u,
                            const void* f, double2* r, int to_f_units, double* d_norms, const Bufs& bufs,
                            cudaStream_t st);
cudaError_t launch_axpy_u(int64_t n, int dtype, const double2* delta, void* u, cudaStream_t st);
// step-5 folds (palindromic global axes), IF offsets, rows x N plane data:
//   forward: plane [rows][N] -> fold [rows][ceil(N/2)] sums, then [rows][floor(N/2)] differences
//   inverse: fold [E | O] -> plane, w_q = E_q + O_q, w_{N-1-q} = E_q - O_q
cudaError_t launch_fold(bool forward, int64_t rows, int N, int64_t plane, int64_t fold, const Bufs& bufs,
                        cudaStream_t st);
// multi-level solve (lfds_ml.cpp) glue:
//   gather: RX[a][k][q] = r[k][q][ifx[a]-1] (all q), RY[b][k][p] = r[k][ify[b]-1][p], 0 at x-interface p
//   lift:   f2[k][y][x] = f[k][y][x] - sigma_k (cL wL[k*ldw+y] [x=0] + cR wR[..] [x=nxc-1]
//                                              + cB wB[k*ldw2+x] [y=0] + cT wT[..] [y=nyc-1])
cudaError_t launch_ml_gather(const double2* r, int nx, int ny, int nz, const int* d_ifx, int nifx, const int* d_ify,
                             int nify, double2* rx, double2* ry, cudaStream_t st);
struct MlLift {
  int nxc, nyc, nz;
  double2 cL, cR, cB, cT;            // face couplings (0 when the face is the outer boundary)
  const double2 *wL, *wR, *wB, *wT;  // w rows on the faces (k-major), or null
  int64_t ldx, ldy;                  // k strides of the x-plane rows (Ny) and y-plane rows (Nx)
  int64_t ox, oy;                    // offsets of the block's first row (y0) / column (x0) in them
};
cudaError_t launch_ml_lift(const MlLift& L, const double2* sig, const double2* f, double2* f2, cudaStream_t st);
// (host) element offsets of RX, RY, WX, WY in a plan's interface buffer and that buffer's byte
// offset in the workspace, for nrhs = 1
struct PlaneLayout {
  int64_t rx, ry, wx, wy;
  size_t off_if;
};
}  // namespace lfds
struct lfds_plan;
namespace lfds {
int plane_layout(lfds_plan* plan, PlaneLayout* out);  // (lfds_host.cpp)
cudaError_t launch_fill_minpiv(double* p, cudaStream_t st);
size_t zsolve_checkpoint_bytes(int nblocks, int max_nx, int max_ny, int R, int nz);
// step 2 with a warp per z-line (lfds_zsolve.cu k_zsw): d_order = owned-block indices grouped by
// class (complex z tables, real tables + complex shift, real tables + real shift), counts[3]
bool zsw_supported(int nz);
cudaError_t launch_zsw(const ZBlock* d_blocks, const int* d_order, const int counts[3], int max_nx, int max_ny, int R,
                       int nz, ZTab tab, const Bufs& bufs, double* d_minpiv, cudaStream_t st);
// resonance margins (lfds_margin.cu): per set, min over (l, m, t) of |ev[lx + l] + ev[ly + m] +
// theta[t]| as a 64-bit key (float bits << 32 | flat index (t * ny + m) * nx + l) in out[set]
struct MarginSet {
  int64_t lx, ly;
  int nx, ny;
};
cudaError_t launch_margins(const double2* d_ev, const MarginSet* d_sets, int nsets, const double2* d_theta, int nz,
                           unsigned long long* d_out, cudaStream_t st);

}  // namespace lfds
