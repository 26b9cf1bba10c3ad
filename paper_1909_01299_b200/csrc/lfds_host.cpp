// Host orchestration and C ABI (include/lfds.h) of the blocked separable solve
// (arXiv 1909.01299).  Setup builds every table once (timed separately);
// lfds_solve enqueues the seven steps as stream-ordered kernels (kernel kinds as reported by
// lfds_kernel_times):
//
//   pass 1 (per block S^ij)   step 1  f~ = (F_x (x) F_y (x) I) f,  F = W^T M
//                                     k_dst2 (uniform x uniform blocks, both axes), k_dstw / k_dst
//                                     (sine x / y passes), k_xform3m / k_xform (dense, complex / real W)
//                             step 2  T_lm v~_lm = f~_lm (z-solves)               k_zs1
//                             step 3  v at the rows next to every block face      k_proj_rows + k_xform3m
//   interface                 step 4  r_b = b - A v on the interface planes       k_iface_res
//                             step 5  w on the planes via the global bases        k_xform3m (plane transforms),
//                                     k_xform (z-modes), k_s5m (modal solve + projections); complex z
//                                     tables: k_zs3 + k_projm
//   pass 2 (per block)        step 6  w~ from the Dirichlet lifting of w          k_xform3m (faces), k_zs2
//                             step 7  u = (W_x (x) W_y (x) I)(v~ + w~), u = w on the planes
//                                     (the step-1 kernels, inverse), k_write_iface
//
// optional refinement: r = M f - A u (k_residual, fp64 or double-double), u += solve(r) (k_axpy).
// k_gemm (plain FP64 tiles) runs only the f64 (real, C1) plans' transforms.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/lfds.h"
#include "lfds_eig.h"
#include "lfds_internal.h"

using namespace lfds;

static thread_local std::string g_err;
static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
#define CUDA_TRY(x)                                                                          \
  do {                                                                                       \
    cudaError_t _e = (x);                                                                    \
    if (_e != cudaSuccess) return fail(LFDS_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

namespace {

// ---- NCCL, loaded at run time (dlopen): the library links no NCCL; the process's own copy
// (the one torch loaded) is preferred.  Only the handful of entry points the exchanges use.
struct NcclId { char internal[128]; };           // == ncclUniqueId
typedef struct ncclComm* NcclComm;                // == ncclComm_t
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(NcclComm*, int, NcclId, int) = nullptr;
  int (*comm_destroy)(NcclComm) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*comm_split)(NcclComm, int, int, NcclComm*, void*) = nullptr;  // optional (NCCL >= 2.18)
  const char* (*error_string)(int) = nullptr;
};
enum { NCCL_FLOAT64 = 8, NCCL_SUM = 0 };
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = nullptr;
  const char* env = getenv("LFDS_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    if (!n) continue;
    h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already in the process (torch)?
    if (!h) h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) return api;
  api.get_unique_id = reinterpret_cast<int (*)(NcclId*)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<int (*)(NcclComm*, int, NcclId, int)>(dlsym(h, "ncclCommInitRank"));
  api.comm_destroy = reinterpret_cast<int (*)(NcclComm)>(dlsym(h, "ncclCommDestroy"));
  api.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t)>(
      dlsym(h, "ncclAllReduce"));
  api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
  api.comm_split = reinterpret_cast<int (*)(NcclComm, int, int, NcclComm*, void*)>(dlsym(h, "ncclCommSplit"));
  api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
  return api;
}

struct AxisBlock {
  int lo, n;         // first node (1-based), interior size
  Basis B;
  int64_t F = 0, W = 0, lam = 0;  // TAB offsets: F[l*n+p] = W[p][l] hh_p, W[p*n+l], lam[l]
  int64_t Fr = -1, Wr = -1;       // real copies (offsets in doubles) when the basis is real (U, R)
  bool dst = false;               // U block with 2(n+1) a supported FFT length: fast sine transform
  double dst_fwd = 0, dst_inv = 0;  // DST-I scale factors sqrt(2h/N), sqrt(2/(hN))
};

struct Axis {
  int N = 0;
  std::vector<zc> h, hh;
  std::vector<int> iface;
  std::vector<AxisBlock> blocks;
  std::vector<int> blk_of;  // per node (0-based): block index or -1 (interface)
  Basis G;                  // global basis
  int64_t Wg = 0, lamg = 0, WI = 0, hoff = 0, hhoff = 0;
  // palindromic steps: every global mode is even or odd under p -> N-1-p (exactly, by the parity
  // split of the eigensolver); the device tables hold the even modes first (ne of them), so the
  // step-5 plane transforms fold the data (x_p +- x_{N-1-p}) and contract half-length (§6a)
  bool gpal = false;
  int ne = 0;
};

// one stage per kernel kind (sine = FFT-based DST on uniform blocks, dense = DMMA contraction)
enum Stage { ST_X1S, ST_X1D, ST_Y1S, ST_Y1D, ST_Z1, ST_EPROJ, ST_EDGE, ST_IFRES, ST_GFWD, ST_GSWEEP, ST_GPROJ,
             ST_GPLANE, ST_FACE, ST_Z2, ST_Y7S, ST_Y7D, ST_X7S, ST_X7D, ST_WRITE, ST_RESID, ST_AXPY, ST_P1S, ST_P7S, ST_P1D, ST_P7D, ST_COUNT };
const char* kStageNames[ST_COUNT] = {
    "step1_x_sine", "step1_x_dense", "step1_y_sine", "step1_y_dense", "step2_zsolve", "step3_edge_projection",
    "step3_edge_values", "step4_iface_residual", "step5_plane_forward", "step5_global_zsolve", "step5_projection",
    "step5_plane_inverse", "step6_face_transform", "step6_zsolve_lift", "step7_y_sine", "step7_y_dense",
    "step7_x_sine", "step7_x_dense", "step7_write_iface", "refine_residual", "refine_axpy", "step1_plane_sine",
    "step7_plane_sine", "step1_plane_dense", "step7_plane_dense"};

// kernel kinds (per-kernel device time: the roofline of the dominant kernel, bench.py)
enum Kern { K_XFORM3M, K_XFORM, K_DSTW, K_DST, K_DST2, K_ZS1, K_ZS2, K_ZS3, K_PROJ, K_PROJM, K_S5M, K_IFRES,
            K_WRITE, K_RESID, K_AXPY, K_GEMM, K_ZSW, K_DSTT, K_FOLD, K_XPLANE, K_COUNT };
const char* kKernNames[K_COUNT] = {
    "k_xform3m", "k_xform", "k_dstw", "k_dst", "k_dst2", "k_zs1", "k_zs2", "k_zs3", "k_proj_rows", "k_projm",
    "k_s5m", "k_iface_res", "k_write_iface", "k_residual", "k_axpy", "k_gemm", "k_zsw", "k_dstt", "k_fold",
    "k_xplane"};

struct Profiler {
  // stage < ST_COUNT: a stage record; stage = ST_COUNT + k: a record of kernel kind k
  struct Rec { int stage, launches; cudaEvent_t a, b; bool graph = false; };  // graph: events owned by a graph
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[ST_COUNT + K_COUNT] = {0};
  int launches[ST_COUNT + K_COUNT] = {0};
  cudaEvent_t get() {
    if (pool.empty()) { cudaEvent_t e; cudaEventCreate(&e); return e; }
    cudaEvent_t e = pool.back(); pool.pop_back(); return e;
  }
};

// Stage-timing event record: inside a stream capture it must be an external event node
// (cudaEventRecordExternal), so that every graph replay re-records it for cudaEventElapsedTime.
static inline void prof_record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else cudaEventRecord(e, st);
}

// experiment knob: LFDS_XPLANE=0 runs the blocks with two small real bases through an x pass and a
// y pass (k_xsmall) instead of the plane transform k_xplane
static int xplane_mode() {  // 0: off; 1 (default): 2-stage ring, 3 CTAs per SM; 4: 3-stage ring, 2 CTAs per SM
  static const int mode = getenv("LFDS_XPLANE") ? atoi(getenv("LFDS_XPLANE")) : 1;
  return mode;
}
static bool xplane_on() { return xplane_mode() != 0; }
// experiment knob: LFDS_XSMALL=0 runs the small real-basis block transforms through k_xform
static bool xsmall_on() {
  static const bool on = !(getenv("LFDS_XSMALL") && atoi(getenv("LFDS_XSMALL")) == 0);
  return on;
}

struct StageDescs {
  int64_t off = 0;  // index of the first desc in the device desc array
  int n = 0, maxM = 0, maxK = 0;
  int64_t maxN = 0;
};

// TMA tensor maps of one strided (y) sine group: one 128-B map per descriptor.  A map embeds the
// address of its input buffer, so every input buffer (i.e. every workspace the plan has solved
// with) gets its own pinned host copy and device copy, encoded once and uploaded stream-ordered
// once; nothing is overwritten afterwards (concurrent solves on other workspaces and captured
// graphs keep reading their own maps)
struct TmaMaps {
  struct Ent {
    void* h = nullptr;       // pinned host maps
    void* d = nullptr;       // device maps
    bool ok = false;
  };
  std::map<const void*, Ent> by_key;  // input buffer -> its maps
};

struct PassPlan {  // descriptors for one (R, in_real, out_real)
  GemmDesc* d_descs = nullptr;
  ZBlock* d_zb = nullptr;
  PDesc* d_pd = nullptr;     // step-3 two-sided edge projections, one per block
  int nzb = 0;               // owned blocks (entries of d_zb before the global one)
  int* d_own = nullptr;      // per-block ownership flags (step-4 partial residual)
  int* d_zwo = nullptr;      // step 2 (k_zsw): owned-block indices grouped by system class
  int zw_cnt[3] = {0, 0, 0}; // blocks per class: complex tables, complex shift, real shift
  int* d_wmask = nullptr;    // block sharding: interface-plane segments this rank writes (k_write_iface)
  int n_pd3 = 0;
  StageDescs s1x, s1y, s3x, s3y, s5r1, s5wx, s6f, s7y, s7x;  // s5r1: R1 and R2; s5wx: WX and WY
  StageDescs s5zf, s5zi;     // z-modal step 5: R~ = Z^T R (R1, R2) and P = Z P~ (P1, P2), real S
  bool s5m = false;          // step 5 in z-modal form (lfds_modal.cu)
  bool fsplit = false;       // formation split of R1~ / R2~ (exchange 3 between phases 2a and 2b)
  int64_t r1t = 0, r2t = 0, p1t = 0, p2t = 0, p2p = 0;
  StageDescs x1c, x1r, y1c, y1r, y7c, y7r, x7c, x7r;  // DMMA transform passes (complex / real S)
  std::vector<std::pair<int, StageDescs>> x1s, y1s, y7s, x7s;  // fast sine transforms, per length n
  std::vector<GemmDesc> h_descs;                                // host copy of d_descs
  std::map<int64_t, TmaMaps> tma;                               // y sine groups (by first descriptor)
  // plane sine transforms of uniform x uniform blocks (k_dst2), per length n: forward (step 1)
  // and inverse (step 7) descriptors in d_dst2 [off, off + count)
  struct Dst2Group { int n; int64_t off; int count; };
  std::vector<Dst2Group> p1s, p7s;
  Dst2Desc* d_dst2 = nullptr;
  // plane transforms of blocks with two bases of at most 32 nodes and no sine form (k_xplane),
  // grouped by the kind of the two matrices (real / complex): forward descriptors of group t in
  // d_xpl[xp_off[t], + xp_cnt[t]), the inverse ones n_xpl further
  XPlaneDesc* d_xpl = nullptr;
  int n_xpl = 0;
  int xp_off[4] = {0, 0, 0, 0}, xp_cnt[4] = {0, 0, 0, 0};  // t = cx + 2 cy
  bool use_xform = false;
  int max_systems = 0, max_systems_global = 0;
  // workspace layout (bytes)
  size_t off_ms = 0, off_t1 = 0, off_if = 0, off_red = 0, off_ck = 0, off_res = 0, total = 0;
  int64_t gp = 0;  // step-5 P1 partials per l-chunk
  int64_t g_off = 0, h_off = 0, vx_off = 0, vy_off = 0, rx = 0, ry = 0, r1 = 0, r2 = 0, p1 = 0, p2 = 0, wx = 0,
          wy = 0, gf = 0, fx = 0, fy = 0;
  bool foldf[2] = {false, false};  // step-5 forward plane transform folded along y (R1) / x (R2)
  bool foldi[2] = {false, false};  // plane inverse folded (unsharded only): WX / WY
};

void free_pass(PassPlan& pp) {
  for (auto& kv : pp.tma)
    for (auto& e : kv.second.by_key) {
      cudaFreeHost(e.second.h);
      cudaFree(e.second.d);
    }
  pp.tma.clear();
  cudaFree(pp.d_descs);
  cudaFree(pp.d_zb);
  cudaFree(pp.d_pd);
  cudaFree(pp.d_own);
  cudaFree(pp.d_wmask);
  cudaFree(pp.d_dst2);
  cudaFree(pp.d_xpl);
  cudaFree(pp.d_zwo);
}

}  // namespace

struct lfds_plan {
  lfds_options opt;
  Axis ax[2];
  int nz = 0;
  std::vector<zc> hz, hhz, sig_node, sig_edge;
  zc lam;
  bool real_z = true;
  int nbx = 0, nby = 0, mpad = 0, lpad = 0, fpad = 0;
  // device tables
  double2* d_tab = nullptr;
  size_t tab_elems = 0;
  ZTab zt_scaled{}, zt_plain{}, zt_lift{};  // zt_lift: zt_scaled rows divided by -sigma_k (step 6)
  std::map<int, int64_t> t_tw;  // FFT twiddle tables per length L
  // step-5 z-modal form (real z tables): Z^T (t x k) and Z (k x t) as real tables (offsets in
  // doubles), theta_t (complex slots)
  bool s5m = false;
  bool xplane_ok = false;  // steps 1 and 7 of the small non-sine blocks as plane transforms (k_xplane)
  int64_t t_zt = 0, t_zf = 0, t_theta = 0;
  int64_t t_dd[3] = {0, 0, 0};  // double-double stencil tables (x, y, z) for the residual
  int64_t t_hz = 0, t_hhz = 0, t_sig = 0, t_sige = 0, t_ifx = 0, t_ify = 0, t_bx = 0, t_by = 0, t_xlo = 0, t_ylo = 0;
  std::map<std::tuple<int, int, int>, PassPlan> passes;
  lfds_report report{};
  lfds_info info{};
  int launches = 0;
  Profiler prof;
  // CUDA graph of the last lfds_solve (options.graph): replayed while the key repeats
  cudaGraphExec_t gexec = nullptr;
  const void* gkey_f = nullptr;
  void* gkey_u = nullptr;
  void* gkey_ws = nullptr;
  size_t gkey_wsb = 0;
  int gkey_nrhs = 0;
  std::vector<Profiler::Rec> grecs;  // stage events captured in the graph (re-recorded per replay)
  lfds_report grep{};
  cudaStream_t cap_stream = nullptr;  // capture happens on a private stream (the legacy default
                                      // stream cannot be captured); the graph runs on the caller's
  // block sharding (lfds_set_partition): owned blocks, the global x-mode range of step 5,
  // and whether this rank adds the b-terms of the interface residual and writes u on the planes
  std::vector<char> own;
  int l_begin = 0, l_end = -1, rank0 = 1;
  int m_begin = 0, m_end = -1;  // z-modal step 5: this rank's global y-modes (-1: all)
  // z-modal step 5, formation split (lfds_set_formation_rows): the rows of R1~ (y-modes) and
  // R2~ (x-modes) this rank FORMS (plane transform + z-transform); exchange 3 sums them over the
  // group that shares them, so every rank's k_s5m still reads its whole (m, l) range (-1: off)
  int fm0 = -1, fm1 = -1, fl0 = -1, fl1 = -1;
  bool sharded = false;
  // in-library exchanges (lfds_set_comm): the NCCL communicator of this rank's group
  NcclComm comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  NcclComm comm_m = nullptr, comm_l = nullptr;  // exchange-3 groups (same y-mode / x-mode range)
  // pivot monitor of the last solve: copied stream-ordered into pinned host memory at its end
  double* h_piv = nullptr;
  cudaStream_t piv_stream = nullptr;
  bool piv_pending = false;
};

namespace {

int64_t align4(int64_t x) { return (x + 3) & ~int64_t(3); }

// ------------------------------------------------------------------ device tables
struct TabBuilder {
  std::vector<double2> v;
  int64_t put(const std::vector<zc>& a) {
    int64_t off = (int64_t)v.size();
    for (auto& z : a) v.push_back(make_double2(z.real(), z.imag()));
    return off;
  }
  int64_t put_real(const std::vector<zc>& a) {  // real parts packed two per slot; offset in doubles
    int64_t off = (int64_t)v.size();
    for (size_t i = 0; i < a.size(); i += 2)
      v.push_back(make_double2(a[i].real(), i + 1 < a.size() ? a[i + 1].real() : 0.0));
    return 2 * off;
  }
  int64_t put_ints(const std::vector<int>& a) {
    int64_t off = (int64_t)v.size();
    size_t slots = (a.size() + 3) / 4;
    v.resize(v.size() + (slots ? slots : 1), make_double2(0, 0));
    if (!a.empty()) std::memcpy(&v[off], a.data(), a.size() * sizeof(int));
    return off;
  }
};

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

GemmDesc gd(int64_t a_off, int64_t sAi, int64_t sAj, int M, int K, int b_buf, int64_t b_off, int64_t sBj, int64_t sB1,
            int64_t sB2, int c_buf, int64_t c_off, int64_t sCi, int64_t sC1, int64_t sC2, int N1, int N2, int flags) {
  GemmDesc d{};
  d.a_off = a_off; d.sAi = sAi; d.sAj = sAj;
  d.b_off = b_off; d.sBj = sBj; d.sB1 = sB1; d.sB2 = sB2;
  d.c_off = c_off; d.sCi = sCi; d.sC1 = sC1; d.sC2 = sC2;
  d.M = M; d.K = K; d.N1 = N1; d.N2 = N2;
  d.b_buf = b_buf; d.c_buf = c_buf; d.flags = flags;
  return d;
}

}  // namespace

// ------------------------------------------------------------------ pass plan (descriptors + workspace layout)
static int build_pass(lfds_plan* P, int R, int in_real, int out_real, PassPlan& pp) {
  const Axis& X = P->ax[0];
  const Axis& Y = P->ax[1];
  const int Nx = X.N, Ny = Y.N, Nz = P->nz;
  const int nbx = P->nbx, nby = P->nby, nblk = nbx * nby;
  const int nifx = (int)X.iface.size(), nify = (int)Y.iface.size();
  // blocks this plan computes (all, unless lfds_set_partition gave this rank a subset)
  auto owned = [&](int b) { return P->own.empty() || P->own[b] != 0; };
  // block mode-space offsets (owned blocks only, packed)
  std::vector<int64_t> ms(nblk, 0), t1(nblk, 0);
  int64_t acc = 0;
  int maxsys = 0;
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      int b = j * nbx + i;
      if (!owned(b)) continue;
      ms[b] = acc;
      t1[b] = acc;
      acc += (int64_t)X.blocks[i].n * Y.blocks[j].n * Nz * R;
      maxsys = std::max(maxsys, X.blocks[i].n * Y.blocks[j].n * R);
    }
  const int64_t ms_elems = acc;
  const int64_t t1_elems = std::max(acc, (int64_t)Nx * Ny * Nz * R);
  // interface buffer layout (complex elements)
  int64_t o = 0;
  pp.g_off = o; o += align4((int64_t)nblk * R * 2 * P->mpad * Nz);
  pp.h_off = o; o += align4((int64_t)nblk * R * 2 * P->lpad * Nz);
  pp.vx_off = o; o += align4((int64_t)nblk * R * 2 * Nz * P->mpad);
  pp.vy_off = o; o += align4((int64_t)nblk * R * 2 * Nz * P->lpad);
  pp.rx = o; o += align4((int64_t)nifx * R * Nz * Ny);
  pp.ry = o; o += align4((int64_t)nify * R * Nz * Nx);
  pp.r1 = o; o += align4((int64_t)nifx * R * Ny * Nz);
  pp.r2 = o; o += align4((int64_t)nify * R * Nx * Nz);
  pp.p1 = o; o += align4((int64_t)nifx * R * Ny * Nz);   // exchange 2 = [p1, p2] (contiguous)
  pp.p2 = o; o += align4((int64_t)nify * R * Nx * Nz);
  pp.gp = o; o += align4((int64_t)(projm_chunks(Nx) > 1 ? projm_chunks(Nx) : 0) * nifx * R * Ny * Nz);
  pp.wx = o; o += align4((int64_t)nifx * R * Nz * Ny);
  pp.wy = o; o += align4((int64_t)nify * R * Nz * Nx);
  pp.gf = o; o += align4((int64_t)nblk * 4 * R * P->fpad * Nz);
  // step-5 fold scratch (palindromic global axes): [sym | anti] halves of the plane data
  pp.fx = o; o += align4((int64_t)nifx * R * Nz * Ny + nifx * R * Nz);
  pp.fy = o; o += align4((int64_t)nify * R * Nz * Nx + nify * R * Nz);
  pp.s5m = P->s5m && !in_real && !out_real && s5m_ka(nifx, nify) > 0;
  if (pp.s5m) {
    pp.r1t = o; o += align4((int64_t)nifx * R * Nz * Ny);
    pp.r2t = o; o += align4((int64_t)nify * R * Nz * Nx);
    pp.p1t = o; o += align4((int64_t)nifx * R * Nz * Ny);
    pp.p2t = o; o += align4((int64_t)nify * R * Nz * Nx);
    pp.p2p = o; o += align4((int64_t)nify * R * Nz * s5m_mtiles(Ny) * Nx);
  }
  const int64_t if_elems = o;
  size_t off = 0;
  // RED (pivot monitor, residual norms) first: the same offset in every pass plan of one R, so
  // the real main pass and the complex refinement pass of an f64 plan share it
  pp.off_red = off; off = al256(off + (size_t)(2 * R + 8) * 8);
  pp.off_ms = off; off = al256(off + ms_elems * 16);
  pp.off_t1 = off; off = al256(off + t1_elems * 16);
  pp.off_if = off; off = al256(off + if_elems * 16);
  pp.off_ck = off;
  off = al256(off + std::max(zsolve_checkpoint_bytes(nblk, P->lpad, P->mpad, R, Nz), zsolve_checkpoint_bytes(1, Nx, Ny, R, Nz)));
  pp.off_res = off;
  if (P->opt.refine != 0) off = al256(off + (size_t)Nx * Ny * Nz * R * 16);
  pp.total = off;
  pp.max_systems = maxsys;

  std::vector<GemmDesc> D;
  auto stage = [&](StageDescs& s, std::vector<GemmDesc>&& v) {
    s.off = (int64_t)D.size();
    s.n = (int)v.size();
    s.maxM = 0;
    s.maxK = 0;
    s.maxN = 0;
    for (auto& d : v) {
      s.maxM = std::max(s.maxM, d.M);
      s.maxK = std::max(s.maxK, d.K);
      s.maxN = std::max(s.maxN, (int64_t)d.N1 * d.N2);
      D.push_back(d);
    }
  };
  const int inF = in_real ? G_BREAL : 0, outF = out_real ? G_CREAL : 0;
  const int64_t RZ = (int64_t)R * Nz;  // merged (r, k) row index
  std::vector<GemmDesc> v;
  // Layouts (complex elements): T1 and MS per block [r][k][q|m][l] (l fastest), so a block's
  // mode space is [rk][m][l] and every z-line (fixed m, l) is strided by nx*ny.
  // step 1: x-forward  T1[rk][q][l] = sum_p F_x[l][p] f[rk][y0+q][x0+p]
  std::vector<int> blk_ids;  // block of each descriptor of the per-block stages s1x, s1y, s7y, s7x
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      blk_ids.push_back(b);
      v.push_back(gd(bx.F, bx.n, 1, bx.n, bx.n, B_F, (int64_t)(by.lo - 1) * Nx + (bx.lo - 1), 1, (int64_t)Nx * Ny, Nx,
                     B_T1, t1[b], 1, (int64_t)by.n * bx.n, bx.n, (int)RZ, by.n, inF));
    }
  stage(pp.s1x, std::move(v)); v.clear();
  //         y-forward  MS[rk][m][l] = sum_q F_y[m][q] T1[rk][q][l]
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      const int64_t pl = (int64_t)bx.n * by.n;
      v.push_back(gd(by.F, by.n, 1, by.n, by.n, B_T1, t1[b], bx.n, pl, 1, B_MS, ms[b], bx.n, pl, 1, (int)RZ, bx.n, 0));
    }
  stage(pp.s1y, std::move(v)); v.clear();
  // step 3 (edge rows G, H of v~): k_proj descriptors below
  // VX[b][e][rk][q] = sum_m W_y[q][m] G[b][e][rk][m];  VY[b][e][rk][p] = sum_l W_x[p][l] H[b][e][rk][l]
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock& by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      v.push_back(gd(by.W, by.n, 1, by.n, by.n, B_IF, pp.g_off + (int64_t)b * 2 * RZ * P->mpad, 1, P->mpad, 0, B_IF,
                     pp.vx_off + (int64_t)b * 2 * RZ * P->mpad, 1, P->mpad, 0, (int)(2 * RZ), 1, 0));
    }
  stage(pp.s3x, std::move(v)); v.clear();
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock& bx = X.blocks[i];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      v.push_back(gd(bx.W, bx.n, 1, bx.n, bx.n, B_IF, pp.h_off + (int64_t)b * 2 * RZ * P->lpad, 1, P->lpad, 0, B_IF,
                     pp.vy_off + (int64_t)b * 2 * RZ * P->lpad, 1, P->lpad, 0, (int)(2 * RZ), 1, 0));
    }
  stage(pp.s3y, std::move(v)); v.clear();
  // step 5: R1[a][rk][m] = sum_q W_y[q][m] RX[a][rk][q];  R2[b][rk][l] = sum_p W_x[p][l] RY[b][rk][p]  (b-units)
  // (both in one launch: the two contractions are independent)
  // (block sharding: step 5 of this rank reads R2[b][rk][l] only for its x-modes l in
  // [l_begin, l_end), so only those rows of W_x^T RY are formed)
  const int l0s = P->sharded ? P->l_begin : 0, l1s = P->sharded ? P->l_end : Nx;
  // (and with a y-mode split of the z-modal step 5, R1 only for the rank's y-modes m)
  const bool msplit = P->sharded && P->m_end >= 0 && P->s5m && !in_real && !out_real;
  const int m0s = msplit ? P->m_begin : 0, m1s = msplit ? P->m_end : Ny;
  // (formation split: this rank forms only its share of those rows, exchange 3 completes them)
  const bool fsplit = P->sharded && P->fm0 >= 0 && P->s5m && !in_real && !out_real;
  const int mf0 = fsplit ? P->fm0 : m0s, mf1 = fsplit ? P->fm1 : m1s;
  const int lf0 = fsplit ? P->fl0 : l0s, lf1 = fsplit ? P->fl1 : l1s;
  pp.fsplit = fsplit;
  // palindromic axis: even modes [0, ne) contract the folded sums x_q + x_{N-1-q} over the first
  // ceil(N/2) rows, odd modes [ne, N) the differences over the first floor(N/2) rows
  auto fwd = [&](const Axis& A, int N, int nif, int64_t src, int64_t fold, int64_t dst, int c0, int c1, bool& folded) {
    if (!nif || c1 <= c0) return;
    const int64_t rows = (int64_t)nif * RZ;
    folded = A.gpal && !in_real && !out_real;
    if (!folded) {
      v.push_back(gd(A.Wg + c0, 1, N, c1 - c0, N, B_IF, src, 1, N, 0, B_IF, dst + c0, 1, N, 0, (int)rows, 1, 0));
      return;
    }
    const int nh = N / 2, ks = N - nh;
    const int e0 = c0, e1 = std::min(c1, A.ne), o0 = std::max(c0, A.ne), o1 = c1;
    if (e1 > e0)
      v.push_back(gd(A.Wg + e0, 1, N, e1 - e0, ks, B_IF, fold, 1, ks, 0, B_IF, dst + e0, 1, N, 0, (int)rows, 1, 0));
    if (o1 > o0 && nh > 0)
      v.push_back(gd(A.Wg + o0, 1, N, o1 - o0, nh, B_IF, fold + rows * ks, 1, nh, 0, B_IF, dst + o0, 1, N, 0, (int)rows,
                     1, 0));
  };
  fwd(Y, Ny, nifx, pp.rx, pp.fx, pp.r1, mf0, mf1, pp.foldf[0]);
  fwd(X, Nx, nify, pp.ry, pp.fy, pp.r2, lf0, lf1, pp.foldf[1]);
  stage(pp.s5r1, std::move(v)); v.clear();
  // P1, P2 (projections of w^ onto the planes): k_projm, see run_pass
  // w on the planes: WX[a][rk][q] = sum_m W_y[q][m] P1[a][rk][m];  WY[b][rk][p] = sum_l W_x[p][l] P2[b][rk][l]
  std::vector<int> wmask;  // sharded: [x-plane a][block row j], then [y-plane b][block column i]
  if (!P->sharded) {
    // palindromic axis: E = W_even P (first ceil(N/2) rows), O = W_odd P (first floor(N/2)
    // rows), then w_q = E_q + O_q and w_{N-1-q} = E_q - O_q (k_unfold)
    auto inv = [&](const Axis& A, int N, int nif, int64_t src, int64_t fold, int64_t dst, bool& folded) {
      if (!nif) return;
      const int64_t rows = (int64_t)nif * RZ;
      folded = A.gpal && !in_real && !out_real;
      if (!folded) {
        v.push_back(gd(A.Wg, N, 1, N, N, B_IF, src, 1, N, 0, B_IF, dst, 1, N, 0, (int)rows, 1, 0));
        return;
      }
      const int nh = N / 2, ks = N - nh;
      v.push_back(gd(A.Wg, N, 1, ks, A.ne, B_IF, src, 1, N, 0, B_IF, fold, 1, ks, 0, (int)rows, 1, 0));
      if (nh > 0 && N - A.ne > 0)
        v.push_back(gd(A.Wg + A.ne, N, 1, nh, N - A.ne, B_IF, src + A.ne, 1, N, 0, B_IF, fold + rows * ks, 1, nh, 0,
                       (int)rows, 1, 0));
    };
    inv(Y, Ny, nifx, pp.p1, pp.fx, pp.wx, pp.foldi[0]);
    inv(X, Nx, nify, pp.p2, pp.fy, pp.wy, pp.foldi[1]);
  } else {
    // Block sharding: a rank needs w on the interface planes only where its own blocks' faces
    // read it (step 6) and where it writes u on the planes (step 7): the segment of x-plane a in
    // block row j belongs to the owner of the block on its left (i = a), the segment of y-plane
    // b in block column i to the owner of the block below (j = b); the plane intersections to
    // rank0.  Only those rows of W_y P1 / W_x P2 are formed.
    auto own_blk = [&](int i, int j) { return owned(j * nbx + i); };
    for (int a = 0; a < nifx; ++a)
      for (int j = 0; j < nby; ++j) {
        const bool writes = own_blk(a, j);
        wmask.push_back(writes ? 1 : 0);
        if (!(writes || own_blk(a + 1, j))) continue;
        const AxisBlock& by = Y.blocks[j];
        v.push_back(gd(Y.Wg + (int64_t)(by.lo - 1) * Ny, Ny, 1, by.n, Ny, B_IF, pp.p1 + (int64_t)a * RZ * Ny, 1, Ny, 0,
                       B_IF, pp.wx + (int64_t)a * RZ * Ny + (by.lo - 1), 1, Ny, 0, (int)RZ, 1, 0));
      }
    for (int b = 0; b < nify; ++b)
      for (int i = 0; i < nbx; ++i) {
        const bool writes = own_blk(i, b);
        wmask.push_back(writes ? 1 : 0);
        if (!(writes || own_blk(i, b + 1))) continue;
        const AxisBlock& bx = X.blocks[i];
        v.push_back(gd(X.Wg + (int64_t)(bx.lo - 1) * Nx, Nx, 1, bx.n, Nx, B_IF, pp.p2 + (int64_t)b * RZ * Nx, 1, Nx, 0,
                       B_IF, pp.wy + (int64_t)b * RZ * Nx + (bx.lo - 1), 1, Nx, 0, (int)RZ, 1, 0));
      }
    if (P->rank0)  // intersections of x-plane a with y-plane b: written from WX[a][rk][q_b]
      // (rows q_b of W_y P1; equally spaced interface rows form one strided descriptor per run,
      // instead of one single-row contraction per intersection)
      for (int a = 0; a < nifx; ++a)
        for (int b0 = 0; b0 < nify;) {
          int cnt = 1;
          const int d = b0 + 1 < nify ? Y.iface[b0 + 1] - Y.iface[b0] : 1;
          while (b0 + cnt < nify && Y.iface[b0 + cnt] - Y.iface[b0 + cnt - 1] == d) ++cnt;
          const int q = Y.iface[b0] - 1;
          v.push_back(gd(Y.Wg + (int64_t)q * Ny, (int64_t)d * Ny, 1, cnt, Ny, B_IF, pp.p1 + (int64_t)a * RZ * Ny, 1, Ny,
                         0, B_IF, pp.wx + (int64_t)a * RZ * Ny + q, d, Ny, 0, (int)RZ, 1, 0));
          b0 += cnt;
        }
  }
  stage(pp.s5wx, std::move(v)); v.clear();
  if (pp.s5m) {  // z-modal step 5: R~[a][r][t][m] = sum_k Z[k][t] R[a][r][k][m]; P = Z P~ (real Z)
    if (nifx && mf1 > mf0)
      v.push_back(gd(P->t_zt, Nz, 1, Nz, Nz, B_IF, pp.r1 + mf0, Ny, (int64_t)Nz * Ny, 1, B_IF, pp.r1t + mf0, Ny,
                     (int64_t)Nz * Ny, 1, nifx * R, mf1 - mf0, 0));
    if (nify && lf1 > lf0)
      v.push_back(gd(P->t_zt, Nz, 1, Nz, Nz, B_IF, pp.r2 + lf0, Nx, (int64_t)Nz * Nx, 1, B_IF, pp.r2t + lf0, Nx,
                     (int64_t)Nz * Nx, 1, nify * R, lf1 - lf0, 0));
    stage(pp.s5zf, std::move(v)); v.clear();
    if (nifx && m1s > m0s)  // (y-mode split: P1 rows outside [m0s, m1s) are zeroed in run_pass)
      v.push_back(gd(P->t_zf, Nz, 1, Nz, Nz, B_IF, pp.p1t + m0s, Ny, (int64_t)Nz * Ny, 1, B_IF, pp.p1 + m0s, Ny,
                     (int64_t)Nz * Ny, 1, nifx * R, m1s - m0s, 0));
    // (block sharding: P2~ is zero outside the rank's x-modes, so only those columns of P2 are
    // formed; run_pass zeroes the rest for the exchange)
    if (nify && l1s > l0s)
      v.push_back(gd(P->t_zf, Nz, 1, Nz, Nz, B_IF, pp.p2t + l0s, Nx, (int64_t)Nz * Nx, 1, B_IF, pp.p2 + l0s, Nx,
                     (int64_t)Nz * Nx, 1, nify * R, l1s - l0s, 0));
    stage(pp.s5zi, std::move(v)); v.clear();
  }
  // step 6: face transforms GF[b][face][rk][mode] (faces L, R, B, T), e.g. GL = F_y w_L
  std::vector<ZBlock> zb;  // owned blocks (k_zs1, k_zs2), then the global 'block' (k_zs3)
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      ZBlock z{};
      z.pad_ = (bx.B.kind != 2 && by.B.kind != 2) ? 1 : 0;  // real eigenvalues: real shift s
      z.ms_off = ms[b];
      z.buf = B_MS;
      z.nx = bx.n;
      z.ny = by.n;
      z.lamx = bx.lam;
      z.lamy = by.lam;
      z.wx0 = bx.W;                                  // row p = 0:   W[0*n + l]
      z.wx1 = bx.W + (int64_t)(bx.n - 1) * bx.n;     // row p = n-1
      z.wy0 = by.W;
      z.wy1 = by.W + (int64_t)(by.n - 1) * by.n;
      z.gL = z.gR = z.gB = z.gT = -1;
      z.fstride = P->fpad;
      z.cL = z.cR = z.cB = z.cT = make_double2(0, 0);
      auto face_off = [&](int face) { return pp.gf + ((int64_t)b * 4 + face) * RZ * P->fpad; };
      const int x1 = bx.lo + bx.n - 1, y1 = by.lo + by.n - 1;
      // x faces: GL[rk][m] = sum_q F_y[m][q] WX[a][rk][y0+q]
      for (int side = 0; side < 2; ++side) {
        if (side == 0 ? i == 0 : i == nbx - 1) continue;
        const int a = side == 0 ? i - 1 : i;
        v.push_back(gd(by.F, by.n, 1, by.n, by.n, B_IF, pp.wx + (int64_t)a * RZ * Ny + (by.lo - 1), 1, Ny, 0, B_IF,
                       face_off(side), 1, P->fpad, 0, (int)RZ, 1, 0));
        zc c = 1.0 / X.h[side == 0 ? bx.lo - 1 : x1];
        if (side == 0) { z.gL = face_off(0); z.cL = make_double2(c.real(), c.imag()); }
        else { z.gR = face_off(1); z.cR = make_double2(c.real(), c.imag()); }
      }
      // y faces: GB[rk][l] = sum_p F_x[l][p] WY[b][rk][x0+p]
      for (int side = 0; side < 2; ++side) {
        if (side == 0 ? j == 0 : j == nby - 1) continue;
        const int bb = side == 0 ? j - 1 : j;
        v.push_back(gd(bx.F, bx.n, 1, bx.n, bx.n, B_IF, pp.wy + (int64_t)bb * RZ * Nx + (bx.lo - 1), 1, Nx, 0, B_IF,
                       face_off(2 + side), 1, P->fpad, 0, (int)RZ, 1, 0));
        zc c = 1.0 / Y.h[side == 0 ? by.lo - 1 : y1];
        if (side == 0) { z.gB = face_off(2); z.cB = make_double2(c.real(), c.imag()); }
        else { z.gT = face_off(3); z.cT = make_double2(c.real(), c.imag()); }
      }
      zb.push_back(z);
    }
  pp.nzb = (int)zb.size();
  {  // step 2 with a warp per line: blocks grouped by class (each class one launch, own registers)
    std::vector<int> ord;
    for (int cls = 0; cls < 3; ++cls) {
      pp.zw_cnt[cls] = 0;
      for (int q = 0; q < pp.nzb; ++q)
        if ((P->real_z ? (zb[q].pad_ ? 2 : 1) : 0) == cls) { ord.push_back(q); ++pp.zw_cnt[cls]; }
    }
    if (!ord.empty()) {
      CUDA_TRY(cudaMalloc(&pp.d_zwo, sizeof(int) * ord.size()));
      CUDA_TRY(cudaMemcpy(pp.d_zwo, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice));
    }
  }
  stage(pp.s6f, std::move(v)); v.clear();
  // step 7: y-inverse T1[rk][q][l] = sum_m W_y[q][m] MS[rk][m][l];  x-inverse u[rk][y0+q][x0+p] = sum_l W_x[p][l] T1
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      const int64_t pl = (int64_t)bx.n * by.n;
      v.push_back(gd(by.W, by.n, 1, by.n, by.n, B_MS, ms[b], bx.n, pl, 1, B_T1, t1[b], bx.n, pl, 1, (int)RZ, bx.n, 0));
    }
  stage(pp.s7y, std::move(v)); v.clear();
  for (int j = 0; j < nby; ++j)
    for (int i = 0; i < nbx; ++i) {
      const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
      int b = j * nbx + i;
      if (!owned(b)) continue;
      v.push_back(gd(bx.W, bx.n, 1, bx.n, bx.n, B_T1, t1[b], 1, (int64_t)by.n * bx.n, bx.n, B_U,
                     (int64_t)(by.lo - 1) * Nx + (bx.lo - 1), 1, (int64_t)Nx * Ny, Nx, (int)RZ, by.n, outF));
    }
  stage(pp.s7x, std::move(v)); v.clear();

  // DMMA transform passes: the same contractions, split by real / complex eigenvector matrix
  pp.use_xform = !in_real && !out_real;
  // blocks uniform on both axes with one length: steps 1 and 7 as plane transforms (k_dst2)
  auto fused2 = [&](int b) {
    const AxisBlock &bx = X.blocks[b % nbx], &by = Y.blocks[b / nbx];
    return P->opt.plane_dst && bx.dst && by.dst && bx.n == by.n && dst2_supported(bx.n);
  };
  // blocks of at most 32 nodes on both axes without a fast sine transform (real or complex
  // bases): steps 1 and 7 as plane transforms (k_xplane)
  auto xplane = [&](int b) {
    const AxisBlock &bx = X.blocks[b % nbx], &by = Y.blocks[b / nbx];
    return P->xplane_ok && !fused2(b) && !bx.dst && !by.dst && bx.n <= 32 && by.n <= 32;
  };
  if (pp.use_xform) {
    std::vector<XPlaneDesc> fw, iv;
    for (int t = 0; t < 4; ++t) {  // groups: t = cx + 2 cy
      pp.xp_off[t] = (int)fw.size();
      for (int b : blk_ids) {
        if (!xplane(b)) continue;
        const AxisBlock &bx = X.blocks[b % nbx], &by = Y.blocks[b / nbx];
        const bool cx = bx.Fr < 0, cy = by.Fr < 0;  // complex matrix: offsets in complex units
        if ((cx ? 1 : 0) + (cy ? 2 : 0) != t) continue;
        const int64_t pl = (int64_t)bx.n * by.n, g0 = (int64_t)(by.lo - 1) * Nx + (bx.lo - 1);
        XPlaneDesc d{};
        d.nx = bx.n; d.ny = by.n; d.nplanes = (int)RZ;
        d.b_buf = B_F; d.b_off = g0; d.sB1 = (int64_t)Nx * Ny; d.sBr = Nx;       // f[rk][y0+q][x0+p]
        d.c_buf = B_MS; d.c_off = ms[b]; d.sC1 = pl; d.sCr = bx.n;                // MS[rk][m][l]
        d.ax = cx ? bx.F : bx.Fr; d.ay = cy ? by.F : by.Fr;
        fw.push_back(d);
        d.b_buf = B_MS; d.b_off = ms[b]; d.sB1 = pl; d.sBr = bx.n;
        d.c_buf = B_U; d.c_off = g0; d.sC1 = (int64_t)Nx * Ny; d.sCr = Nx;        // u[rk][y0+q][x0+p]
        d.ax = cx ? bx.W : bx.Wr; d.ay = cy ? by.W : by.Wr;
        iv.push_back(d);
      }
      pp.xp_cnt[t] = (int)fw.size() - pp.xp_off[t];
    }
    pp.n_xpl = (int)fw.size();
    if (pp.n_xpl) {
      fw.insert(fw.end(), iv.begin(), iv.end());
      CUDA_TRY(cudaMalloc(&pp.d_xpl, sizeof(XPlaneDesc) * fw.size()));
      CUDA_TRY(cudaMemcpy(pp.d_xpl, fw.data(), sizeof(XPlaneDesc) * fw.size(), cudaMemcpyHostToDevice));
    }
  }
  if (pp.use_xform) {
    std::map<int, std::vector<Dst2Desc>> f2, i2;  // per length n
    for (int b : blk_ids) {
      if (!fused2(b)) continue;
      const AxisBlock &bx = X.blocks[b % nbx], &by = Y.blocks[b / nbx];
      const int64_t pl = (int64_t)bx.n * by.n, g0 = (int64_t)(by.lo - 1) * Nx + (bx.lo - 1);
      Dst2Desc d{};
      d.tw_off = P->t_tw.at(2 * (bx.n + 1));
      d.nplanes = (int)RZ;
      d.b_buf = B_F; d.b_off = g0; d.sB1 = (int64_t)Nx * Ny; d.sBr = Nx;       // f[rk][y0+q][x0+p]
      d.c_buf = B_MS; d.c_off = ms[b]; d.sC1 = pl; d.sCr = bx.n;                // MS[rk][m][l]
      d.ax = bx.dst_fwd; d.ay = by.dst_fwd;
      f2[bx.n].push_back(d);
      d.b_buf = B_MS; d.b_off = ms[b]; d.sB1 = pl; d.sBr = bx.n;                // MS[rk][m][l]
      d.c_buf = B_U; d.c_off = g0; d.sC1 = (int64_t)Nx * Ny; d.sCr = Nx;        // u[rk][y0+q][x0+p]
      d.ax = bx.dst_inv; d.ay = by.dst_inv;
      i2[bx.n].push_back(d);
    }
    std::vector<Dst2Desc> all;
    for (auto* m : {&f2, &i2})
      for (auto& kv : *m) {
        (m == &f2 ? pp.p1s : pp.p7s).push_back({kv.first, (int64_t)all.size(), (int)kv.second.size()});
        all.insert(all.end(), kv.second.begin(), kv.second.end());
      }
    if (!all.empty()) {
      CUDA_TRY(cudaMalloc(&pp.d_dst2, sizeof(Dst2Desc) * all.size()));
      CUDA_TRY(cudaMemcpy(pp.d_dst2, all.data(), sizeof(Dst2Desc) * all.size(), cudaMemcpyHostToDevice));
    }
  }
  if (pp.use_xform) {
    std::vector<GemmDesc> vc, vr;
    auto split = [&](StageDescs& sc, StageDescs& sr, std::vector<std::pair<int, StageDescs>>& sd,
                     const StageDescs& src, bool xaxis, bool fwd) {
      std::map<int, std::vector<GemmDesc>> vd;  // DST descriptors grouped by block length
      for (int q = 0; q < src.n; ++q) {
        GemmDesc d = D[src.off + q];
        // stages s1x/s7x/s1y/s7y hold one descriptor per owned block, in block order
        const int b = blk_ids[q];
        const AxisBlock& ab = xaxis ? X.blocks[b % nbx] : Y.blocks[b / nbx];
        const int64_t roff = fwd ? ab.Fr : ab.Wr;
        if (fused2(b) || xplane(b)) continue;  // k_dst2 / k_xplane (both axes at once)
        if (ab.dst) {
          d.scale = fwd ? ab.dst_fwd : ab.dst_inv;
          d.a_off = P->t_tw.at(2 * (ab.n + 1));  // twiddles W_L^j of the odd-extension FFT
          vd[ab.n].push_back(d);
        }
        else if (roff >= 0) { d.a_off = roff; vr.push_back(d); }
        else vc.push_back(d);
      }
      stage(sc, std::move(vc)); vc.clear();
      stage(sr, std::move(vr)); vr.clear();
      for (auto& kv : vd) {
        StageDescs t;
        stage(t, std::move(kv.second));
        sd.emplace_back(kv.first, t);
      }
    };
    split(pp.x1c, pp.x1r, pp.x1s, pp.s1x, true, true);
    split(pp.y1c, pp.y1r, pp.y1s, pp.s1y, false, true);
    split(pp.y7c, pp.y7r, pp.y7s, pp.s7y, false, false);
    split(pp.x7c, pp.x7r, pp.x7s, pp.s7x, true, false);
  }

  pp.h_descs = D;
  CUDA_TRY(cudaMalloc(&pp.d_descs, sizeof(GemmDesc) * std::max<size_t>(1, D.size())));
  CUDA_TRY(cudaMemcpy(pp.d_descs, D.data(), sizeof(GemmDesc) * D.size(), cudaMemcpyHostToDevice));
  {  // the step-5 global z-solve as one more 'block': all Nx x Ny global modes, in place in T1
    ZBlock g{};
    g.ms_off = 0;
    g.buf = B_T1;
    g.nx = Nx;
    g.ny = Ny;
    g.lamx = X.lamg;
    g.lamy = Y.lamg;
    g.pad_ = (X.G.kind != 2 && Y.G.kind != 2) ? 1 : 0;
    g.gL = g.gR = g.gB = g.gT = -1;
    zb.push_back(g);
    pp.max_systems_global = Nx * Ny * R;
  }
  {  // step 3: G = (edge rows of W_x) v~, H = (edge rows of W_y) v~, one read of v~ per block
    std::vector<PDesc> pd;
    for (int j = 0; j < nby; ++j)
      for (int i = 0; i < nbx; ++i) {
        const AxisBlock &bx = X.blocks[i], &by = Y.blocks[j];
        const int b = j * nbx + i;
        if (!owned(b)) continue;
        PDesc d{};
        d.x_off = ms[b];
        d.ps = (int64_t)bx.n * by.n;
        d.x_buf = B_MS;
        d.nx = bx.n;
        d.ny = by.n;
        d.nplanes = (int)RZ;
        d.E1 = d.E2 = 2;
        d.wr = bx.W;                                 // rows p = 0 and p = n-1 of W_x
        d.wr_es = (int64_t)(bx.n - 1) * bx.n;
        d.wc = by.W;
        d.wc_es = (int64_t)(by.n - 1) * by.n;
        d.g_off = pp.g_off + (int64_t)b * 2 * RZ * P->mpad;  // G[b][e][rk][m]
        d.g_es = RZ * P->mpad;
        d.g_ps = P->mpad;
        d.h_off = pp.h_off + (int64_t)b * 2 * RZ * P->lpad;  // H[b][e][rk][l]
        d.h_es = RZ * P->lpad;
        d.h_ps = P->lpad;
        pd.push_back(d);
      }
    pp.n_pd3 = (int)pd.size();
    CUDA_TRY(cudaMalloc(&pp.d_pd, sizeof(PDesc) * std::max<size_t>(1, pd.size())));
    CUDA_TRY(cudaMemcpy(pp.d_pd, pd.data(), sizeof(PDesc) * pd.size(), cudaMemcpyHostToDevice));
  }
  {
    std::vector<int> own(nblk);
    for (int b = 0; b < nblk; ++b) own[b] = owned(b) ? 1 : 0;
    CUDA_TRY(cudaMalloc(&pp.d_own, sizeof(int) * nblk));
    CUDA_TRY(cudaMemcpy(pp.d_own, own.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice));
    if (!wmask.empty()) {
      CUDA_TRY(cudaMalloc(&pp.d_wmask, sizeof(int) * wmask.size()));
      CUDA_TRY(cudaMemcpy(pp.d_wmask, wmask.data(), sizeof(int) * wmask.size(), cudaMemcpyHostToDevice));
    }
  }
  CUDA_TRY(cudaMalloc(&pp.d_zb, sizeof(ZBlock) * zb.size()));
  CUDA_TRY(cudaMemcpy(pp.d_zb, zb.data(), sizeof(ZBlock) * zb.size(), cudaMemcpyHostToDevice));
  return LFDS_OK;
}

static int get_pass(lfds_plan* P, int R, int in_real, int out_real, PassPlan** out) {
  auto key = std::make_tuple(R, in_real, out_real);
  auto it = P->passes.find(key);
  if (it == P->passes.end()) {
    PassPlan pp;
    int rc = build_pass(P, R, in_real, out_real, pp);
    if (rc) return rc;
    it = P->passes.emplace(key, pp).first;
  }
  *out = &it->second;
  return LFDS_OK;
}

// ------------------------------------------------------------------ one pipeline pass (steps 1-7)
// phases (bit mask): 1 = pass 1 (steps 1-3) and this rank's part of the step-4 residual;
// 2 = step 5 on this rank's global x-modes; 4 = plane inverse, pass 2 (steps 6-7).  With block
// sharding the caller sums exchange 1 ([RX, RY]) over the ranks between phases 1 and 2 and
// exchange 2 ([P1, P2]) between phases 2 and 4 (lfds_exchange_layout).
enum { PH_1 = 1, PH_2A = 2, PH_3 = 4, PH_2B = 8, PH_2 = PH_2A | PH_2B, PH_ALL = 15, PH_INV = 16 };
static int run_pass(lfds_plan* P, PassPlan& pp, Bufs bufs, int R, int in_dtype, int out_dtype, cudaStream_t st,
                    int phases = PH_ALL) {
  const Axis& X = P->ax[0];
  const Axis& Y = P->ax[1];
  const int Nx = X.N, Ny = Y.N, Nz = P->nz;
  const int nifx = (int)X.iface.size(), nify = (int)Y.iface.size();
  const int nblk = P->nbx * P->nby;
  double* minpiv = reinterpret_cast<double*>(bufs.p[B_RED]);
  const bool prof = P->opt.profile != 0;
  const bool kprof = P->opt.profile >= 2;  // per-kernel-kind events too
  int cur_stage = -1, cur_launch0 = 0;
  cudaEvent_t ev_a = nullptr;
  auto begin = [&](int stg) {
    cur_stage = stg;
    cur_launch0 = P->launches;
    if (prof) { ev_a = P->prof.get(); prof_record(ev_a, st); }
  };
  auto end = [&]() {
    if (prof && cur_stage >= 0) {
      cudaEvent_t b = P->prof.get();
      prof_record(b, st);
      P->prof.recs.push_back({cur_stage, P->launches - cur_launch0, ev_a, b});
    }
    cur_stage = -1;
  };
  // kernel-kind events (inside the stage events): device time per kernel kind, `n` launches
  auto kern = [&](int k, int n, auto&& launch) -> cudaError_t {
    cudaEvent_t a = nullptr;
    if (kprof) { a = P->prof.get(); prof_record(a, st); }
    const cudaError_t e = launch();
    P->launches += n;
    if (kprof) {
      cudaEvent_t b = P->prof.get();
      prof_record(b, st);
      P->prof.recs.push_back({ST_COUNT + k, n, a, b});
    }
    return e;
  };
  auto nl = [](int ndesc) { return (ndesc + 65534) / 65535; };
  auto gemm = [&](const StageDescs& s) -> int {
    if (!s.n) return LFDS_OK;
    CUDA_TRY(kern(K_GEMM, nl(s.n), [&] {
      return launch_gemm(pp.d_descs + s.off, s.n, s.maxM, (int)std::min<int64_t>(s.maxN, INT32_MAX), 0, bufs, st); }));
    return LFDS_OK;
  };
  // transform pass: sine-transform launches timed as stage st_s, dense ones as st_d
  auto xform = [&](const StageDescs& sc, const StageDescs& sr, const StageDescs& generic, bool kcontig,
                   const std::vector<std::pair<int, StageDescs>>* sd, int st_s, int st_d) -> int {
    if (!pp.use_xform) {
      begin(st_d);
      int r = gemm(generic);
      end();
      return r;
    }
    if (sd && !sd->empty()) {
      begin(st_s);
      for (auto& kv : *sd) {
        // strided (y) passes: TMA-fed tiles when the maps can be built for this input buffer
        if (!kcontig && P->opt.dst_tma && dst_tma_supported(kv.first)) {
          const GemmDesc* hd = pp.h_descs.data() + kv.second.off;
          const void* key = bufs.p[hd[0].b_buf];
          auto found = pp.tma[kv.second.off].by_key.find(key);
          if (found == pp.tma[kv.second.off].by_key.end()) {
            TmaMaps::Ent e;
            const size_t nb = (size_t)kv.second.n * 128;
            CUDA_TRY(cudaMallocHost(&e.h, nb));
            CUDA_TRY(cudaMalloc(&e.d, nb));
            e.ok = true;
            for (int q = 0; q < kv.second.n && e.ok; ++q)
              e.ok = dst_tma_encode(hd[q], kv.first, bufs, static_cast<char*>(e.h) + (size_t)q * 128);
            if (e.ok) CUDA_TRY(cudaMemcpyAsync(e.d, e.h, nb, cudaMemcpyHostToDevice, st));
            found = pp.tma[kv.second.off].by_key.emplace(key, e).first;
          }
          const TmaMaps::Ent& tm = found->second;
          if (tm.ok) {
            int maxN1 = 0, maxN2 = 0;
            for (int q = 0; q < kv.second.n; ++q) { maxN1 = std::max(maxN1, hd[q].N1); maxN2 = std::max(maxN2, hd[q].N2); }
            CUDA_TRY(kern(K_DSTT, 1, [&] {
              return launch_dst_tma(pp.d_descs + kv.second.off, tm.d, kv.second.n, kv.first, maxN2, maxN1, bufs, st); }));
            continue;
          }
        }
        CUDA_TRY(kern(kcontig ? K_DSTW : K_DST, nl(kv.second.n), [&] {
          return launch_dst(pp.d_descs + kv.second.off, kv.second.n, kv.first, kv.second.maxN, kcontig, bufs, st); }));
      }
      end();
    }
    begin(st_d);
    if (sc.n)
      CUDA_TRY(kern(K_XFORM3M, nl(sc.n), [&] {
        return launch_xform(pp.d_descs + sc.off, sc.n, sc.maxM, sc.maxN, false, kcontig, bufs, st); }));
    if (sr.n)
      CUDA_TRY(kern(K_XFORM, nl(sr.n), [&] {
        if (sr.maxM <= 32 && sr.maxK <= 32 && xsmall_on())
          return launch_xform_small(pp.d_descs + sr.off, sr.n, sr.maxK, sr.maxN, kcontig, bufs, st);
        return launch_xform(pp.d_descs + sr.off, sr.n, sr.maxM, sr.maxN, true, kcontig, bufs, st); }));
    end();
    return LFDS_OK;
  };
  // plane sine transforms (uniform x uniform blocks), one launch per block length
  // plane transforms of the blocks with two small real bases (k_xplane)
  auto planex = [&](bool fwd) -> int {
    if (!pp.n_xpl) return LFDS_OK;
    begin(fwd ? ST_P1D : ST_P7D);
    for (int t = 0; t < 4; ++t)
      if (pp.xp_cnt[t])
        CUDA_TRY(kern(K_XPLANE, nl(pp.xp_cnt[t]), [&] {
          return launch_xplane(pp.d_xpl + (fwd ? 0 : pp.n_xpl) + pp.xp_off[t], pp.xp_cnt[t], (int)((int64_t)R * Nz),
                               bufs, st, xplane_mode(), (t & 1) != 0, (t & 2) != 0); }));
    end();
    return LFDS_OK;
  };
  auto plane2 = [&](const std::vector<PassPlan::Dst2Group>& gs, int stg) -> int {
    if (gs.empty()) return LFDS_OK;
    begin(stg);
    for (auto& g : gs)
      CUDA_TRY(kern(K_DST2, nl(g.count), [&] {
        return launch_dst2(pp.d_dst2 + g.off, g.count, g.n, (int)((int64_t)R * Nz), bufs, st); }));
    end();
    return LFDS_OK;
  };
  // step-5 plane data folded for the half-length contractions of palindromic global axes:
  // forward (before the plane transform) x -> [x_q + x_{N-1-q} | x_q - x_{N-1-q}]; inverse (after)
  // [E | O] -> w_q = E_q + O_q, w_{N-1-q} = E_q - O_q
  auto fold_planes = [&](bool forward) -> int {
    const bool* fl = forward ? pp.foldf : pp.foldi;
    if (!fl[0] && !fl[1]) return LFDS_OK;
    if (prof) begin(forward ? ST_GFWD : ST_GPLANE);
    for (int ax = 0; ax < 2; ++ax) {
      if (!fl[ax]) continue;
      const int N = ax == 0 ? Ny : Nx;
      const int64_t rows = (int64_t)(ax == 0 ? nifx : nify) * R * Nz;
      const int64_t plane = ax == 0 ? (forward ? pp.rx : pp.wx) : (forward ? pp.ry : pp.wy);
      const int64_t fold = ax == 0 ? pp.fx : pp.fy;
      CUDA_TRY(kern(K_FOLD, 1, [&] { return launch_fold(forward, rows, N, plane, fold, bufs, st); }));
    }
    if (prof) end();
    return LFDS_OK;
  };
  int rc;
  const bool has_if = nifx + nify > 0;
  const int l_begin = P->sharded ? P->l_begin : 0, l_end = P->sharded ? P->l_end : Nx;
  (void)nblk;
  // pass 1
  if (phases & PH_1) {
  if ((rc = plane2(pp.p1s, ST_P1S))) return rc;
  if ((rc = planex(true))) return rc;
  if ((rc = xform(pp.x1c, pp.x1r, pp.s1x, true, &pp.x1s, ST_X1S, ST_X1D))) return rc;
  if ((rc = xform(pp.y1c, pp.y1r, pp.s1y, false, &pp.y1s, ST_Y1S, ST_Y1D))) return rc;
  begin(ST_Z1);
  if (pp.nzb && P->opt.zs_warp && zsw_supported(Nz))  // a warp per z-line, one read and one write of v~
    CUDA_TRY(kern(K_ZSW, (pp.zw_cnt[0] > 0) + (pp.zw_cnt[1] > 0) + (pp.zw_cnt[2] > 0), [&] {
      return launch_zsw(pp.d_zb, pp.d_zwo, pp.zw_cnt, P->lpad, P->mpad, R, Nz, P->zt_scaled, bufs, minpiv, st); }));
  else if (pp.nzb)
    CUDA_TRY(kern(K_ZS1, 1, [&] {
      return launch_zsolve(1, pp.d_zb, pp.nzb, P->lpad, P->mpad, R, Nz, P->zt_scaled, P->t_sig, nullptr, bufs, minpiv,
                           st, P->real_z); }));
  end();
  if (has_if) {
    begin(ST_EPROJ);
    CUDA_TRY(kern(K_PROJ, 1, [&] { return launch_proj(pp.d_pd, pp.n_pd3, P->lpad, 2, R * Nz, st, bufs); }));
    end(); begin(ST_EDGE);
    // node values next to the faces: VX = W_y G, VY = W_x H (DMMA, complex path)
    if (pp.use_xform) {
      for (const StageDescs* s3 : {&pp.s3x, &pp.s3y})
        if (s3->n)
          CUDA_TRY(kern(K_XFORM3M, nl(s3->n), [&] {
            return launch_xform(pp.d_descs + s3->off, s3->n, s3->maxM, s3->maxN, false, true, bufs, st); }));
    } else {
      if ((rc = gemm(pp.s3x))) return rc;
      if ((rc = gemm(pp.s3y))) return rc;
    }
    end(); begin(ST_IFRES);
    // step 4
    IfaceRes ir{};
    ir.nx = Nx; ir.ny = Ny; ir.nz = Nz; ir.R = R; ir.nifx = nifx; ir.nify = nify; ir.dtype = in_dtype;
    ir.ifx = P->t_ifx; ir.ify = P->t_ify;
    ir.hx = X.hoff; ir.hy = Y.hoff; ir.hhx = X.hhoff; ir.hhy = Y.hhoff; ir.hhz = P->t_hhz; ir.sig = P->t_sig;
    ir.rx = pp.rx; ir.ry = pp.ry; ir.vxo = pp.vx_off; ir.vyo = pp.vy_off;
    ir.blk_of_x = P->t_bx; ir.blk_of_y = P->t_by; ir.xlo = P->t_xlo; ir.ylo = P->t_ylo;
    ir.nbx = P->nbx; ir.nby = P->nby; ir.qpad = P->mpad; ir.ppad = P->lpad;
    ir.own = pp.d_own; ir.with_b = P->sharded ? P->rank0 : 1;
    CUDA_TRY(kern(K_IFRES, 1, [&] { return launch_iface_residual(ir, bufs, st); }));
    end();
  }
  }
  if ((phases & PH_2A) && has_if && pp.s5m) {
    // step 5, z-modal form: plane transforms (W_y^T, W_x^T), z-modes (Z^T), the modal solve
    // projected onto the planes, back to z (Z) -> exchange 2 = [P1, P2]
    if (pp.fsplit)  // formation split: rows this rank does not form are zero in exchange 3
      CUDA_TRY(cudaMemsetAsync(reinterpret_cast<double2*>(bufs.p[B_IF]) + pp.r1t, 0,
                               sizeof(double2) * (size_t)(pp.p1t - pp.r1t), st));
    if ((rc = fold_planes(true))) return rc;
    if ((rc = xform(pp.s5r1, StageDescs{}, pp.s5r1, true, nullptr, ST_GFWD, ST_GFWD))) return rc;
    begin(ST_GFWD);
    if (pp.s5zf.n)
      CUDA_TRY(kern(K_XFORM, 1, [&] {
        return launch_xform(pp.d_descs + pp.s5zf.off, pp.s5zf.n, pp.s5zf.maxM, pp.s5zf.maxN, true, false, bufs, st); }));
    end();
  }
  if ((phases & PH_2B) && has_if && pp.s5m) {
    begin(ST_GSWEEP);
    S5M S{};
    S.nx = Nx; S.ny = Ny; S.nz = Nz; S.R = R; S.nifx = nifx; S.nify = nify;
    S.l_begin = l_begin; S.l_end = l_end; S.nmt = s5m_mtiles(Ny);
    const bool msplit = P->sharded && P->m_end >= 0;
    S.mt_begin = msplit ? (P->m_begin + 63) / 64 : 0;  // (an empty range at the end: [ny, ny))
    S.mt_end = msplit ? (P->m_end + 63) / 64 : S.nmt;
    S.lamx = X.lamg; S.lamy = Y.lamg; S.theta = P->t_theta; S.wxi = X.WI; S.wyi = Y.WI;
    S.r1t = pp.r1t; S.r2t = pp.r2t; S.p1t = pp.p1t; S.p2p = pp.p2p; S.p2t = pp.p2t;
    CUDA_TRY(kern(K_S5M, nify ? 2 : 1, [&] { return launch_s5m(S, bufs, st); }));
    end(); begin(ST_GPROJ);
    if (msplit && nifx)  // P1 rows of other y-modes: zero (exchange 2 sums the ranks' parts)
      CUDA_TRY(cudaMemsetAsync(reinterpret_cast<double2*>(bufs.p[B_IF]) + pp.p1, 0,
                               sizeof(double2) * (size_t)nifx * R * Nz * Ny, st));
    if (P->sharded && nify && (l_begin > 0 || l_end < Nx))  // P2 columns of other x-modes: zero
      CUDA_TRY(cudaMemsetAsync(reinterpret_cast<double2*>(bufs.p[B_IF]) + pp.p2, 0,
                               sizeof(double2) * (size_t)nify * R * Nz * Nx, st));
    if (pp.s5zi.n)
      CUDA_TRY(kern(K_XFORM, 1, [&] {
        return launch_xform(pp.d_descs + pp.s5zi.off, pp.s5zi.n, pp.s5zi.maxM, pp.s5zi.maxN, true, false, bufs, st); }));
    end();
  } else if ((phases & PH_2A) && has_if && !pp.s5m) {
    // step 5
    if ((rc = fold_planes(true))) return rc;
    if ((rc = xform(pp.s5r1, StageDescs{}, pp.s5r1, true, nullptr, ST_GFWD, ST_GFWD))) return rc;
    begin(ST_GSWEEP);
    GSweep g{};
    g.nx = Nx; g.ny = Ny; g.nifx = nifx; g.nify = nify; g.nz = Nz; g.R = R;
    g.lamx = X.lamg; g.lamy = Y.lamg; g.wxi = X.WI; g.wyi = Y.WI; g.r1 = pp.r1; g.r2 = pp.r2; g.what = 0;
    g.l_begin = l_begin; g.l_end = l_end;
    CUDA_TRY(kern(K_ZS3, 1, [&] {
      return launch_zsolve(3, pp.d_zb + pp.nzb, 1, Nx, Ny, R, Nz, P->zt_plain, P->t_sig, &g, bufs, minpiv, st,
                           P->real_z); }));
    end(); begin(ST_GPROJ);
    {
      const int64_t RZ = (int64_t)R * Nz;
      if (l_begin >= l_end) {  // no x-modes on this rank: it contributes zero to exchange 2
        CUDA_TRY(cudaMemsetAsync(reinterpret_cast<double2*>(bufs.p[B_IF]) + pp.p1, 0,
                                 sizeof(double2) * (size_t)(pp.gp - pp.p1), st));
      } else if (l_begin > 0 || l_end < Nx) {  // P2 rows outside this rank's x-modes must sum to zero
        CUDA_TRY(cudaMemsetAsync(reinterpret_cast<double2*>(bufs.p[B_IF]) + pp.p2, 0,
                                 sizeof(double2) * (size_t)nify * RZ * Nx, st));
      }
      ProjM pm{};
      pm.nx = Nx; pm.ny = Ny; pm.nplanes = R * Nz; pm.E1 = nifx; pm.E2 = nify;
      pm.l_begin = l_begin; pm.l_end = l_end; pm.nlc = projm_chunks(l_end - l_begin);
      pm.x_buf = B_T1; pm.x_off = 0; pm.wr = X.WI; pm.wc = Y.WI;
      pm.g_es = RZ * Ny; pm.g_ps = Ny; pm.p1_off = pp.p1; pm.p1_es = RZ * Ny;
      if (pm.nlc > 1) { pm.g_off = pp.gp; pm.g_lcs = (int64_t)nifx * RZ * Ny; }
      else { pm.g_off = pp.p1; pm.g_lcs = 0; }
      pm.h_off = pp.p2; pm.h_es = RZ * Nx; pm.h_ps = Nx;
      CUDA_TRY(kern(K_PROJM, pm.nlc > 1 ? 2 : 1, [&] { return launch_projm(pm, bufs, st); }));
    }
    end();
  }
  if ((phases & PH_INV) && has_if) {
    // w on the interface planes only (the multi-level solve's coarse level): plane inverse and
    // u = w on the planes, no block pass
    if ((rc = xform(pp.s5wx, StageDescs{}, pp.s5wx, true, nullptr, ST_GPLANE, ST_GPLANE))) return rc;
    if ((rc = fold_planes(false))) return rc;
    begin(ST_WRITE);
    CUDA_TRY(kern(K_WRITE, 1, [&] {
      return launch_write_iface_u(Nx, Ny, Nz, R, out_dtype, nifx, nify, P->t_ifx, P->t_ify, pp.wx, pp.wy, bufs, st,
                                  pp.d_wmask, P->t_bx, P->t_by, P->nbx, P->nby, P->sharded ? P->rank0 : 1); }));
    end();
  }
  if (phases & PH_3) {
  if (has_if) {
    if ((rc = xform(pp.s5wx, StageDescs{}, pp.s5wx, true, nullptr, ST_GPLANE, ST_GPLANE))) return rc;
    if ((rc = fold_planes(false))) return rc;
    begin(ST_FACE);
    // step 6: face transforms (DMMA, complex path)
    if (pp.use_xform && pp.s6f.n) {
      CUDA_TRY(kern(K_XFORM3M, nl(pp.s6f.n), [&] {
        return launch_xform(pp.d_descs + pp.s6f.off, pp.s6f.n, pp.s6f.maxM, pp.s6f.maxN, false, true, bufs, st); }));
    } else if ((rc = gemm(pp.s6f))) {
      return rc;
    }
    end(); begin(ST_Z2);
    if (pp.nzb)
      CUDA_TRY(kern(K_ZS2, 1, [&] {
        return launch_zsolve(2, pp.d_zb, pp.nzb, P->lpad, P->mpad, R, Nz, P->zt_lift, P->t_sig, nullptr, bufs, minpiv,
                             st, P->real_z); }));
    end();
  }
  // step 7
  if ((rc = plane2(pp.p7s, ST_P7S))) return rc;
  if ((rc = planex(false))) return rc;
  if ((rc = xform(pp.y7c, pp.y7r, pp.s7y, false, &pp.y7s, ST_Y7S, ST_Y7D))) return rc;
  if ((rc = xform(pp.x7c, pp.x7r, pp.s7x, true, &pp.x7s, ST_X7S, ST_X7D))) return rc;
  if (has_if) {  // (sharded: every rank writes its own segments of the planes, pp.d_wmask)
    begin(ST_WRITE);
    CUDA_TRY(kern(K_WRITE, 1, [&] {
      return launch_write_iface_u(Nx, Ny, Nz, R, out_dtype, nifx, nify, P->t_ifx, P->t_ify, pp.wx, pp.wy, bufs, st,
                                  pp.d_wmask, P->t_bx, P->t_by, P->nbx, P->nby, P->sharded ? P->rank0 : 1); }));
    end();
  }
  }
  return LFDS_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

void lfds_default_options(lfds_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->dtype = LFDS_C128;
  o->refine = 0;
  o->refine_tol = 1e-13;
  o->residual_dd = 1;
  o->device = 0;
  o->rhs_chunk = 0;
  o->profile = 0;
  o->s5_modal = 1;
  o->graph = 0;
  o->plane_dst = 1;
  o->resonance_tol = 1e-13;
  o->zs_warp = 0;
  o->dst_tma = 1;
}

int lfds_stage_count(void) { return ST_COUNT; }
const char* lfds_stage_name(int i) { return (i >= 0 && i < ST_COUNT) ? kStageNames[i] : ""; }

// accumulate the pending stage records (waits for their events)
static int prof_drain(lfds_plan* P);
// the captured graph replays launches that read the pass plans' device descriptors and the
// workspace layout they were built for: drop it whenever the pass plans are freed
static void drop_graph(lfds_plan* P) {
  if (!P->gexec) return;
  prof_drain(P);  // pending replay records refer to the graph's events
  cudaGraphExecDestroy(P->gexec);
  P->gexec = nullptr;
  for (auto& r : P->grecs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  P->grecs.clear();
  P->gkey_f = nullptr; P->gkey_u = nullptr; P->gkey_ws = nullptr; P->gkey_wsb = 0; P->gkey_nrhs = 0;
}

static int prof_drain(lfds_plan* P) {
  for (auto& r : P->prof.recs) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    P->prof.ms[r.stage] += t;
    P->prof.launches[r.stage] += r.launches;
    if (!r.graph) {
      P->prof.pool.push_back(r.a);
      P->prof.pool.push_back(r.b);
    }
  }
  P->prof.recs.clear();
  return LFDS_OK;
}

int lfds_stage_times(lfds_plan* P, double* ms, int* launches) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  int rc;
  if ((rc = prof_drain(P))) return rc;
  for (int i = 0; i < ST_COUNT; ++i) {
    if (ms) ms[i] = P->prof.ms[i];
    if (launches) launches[i] = P->prof.launches[i];
    P->prof.ms[i] = 0;
    P->prof.launches[i] = 0;
  }
  return LFDS_OK;
}

int lfds_set_profile(lfds_plan* P, int level) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (level < 0 || level > 2) return fail(LFDS_EINVAL, "profile level must be 0, 1 or 2");
  if (level != P->opt.profile) drop_graph(P);  // the captured graph holds the old event nodes
  P->opt.profile = level;
  return LFDS_OK;
}

int lfds_kernel_count(void) { return K_COUNT; }
const char* lfds_kernel_name(int i) { return (i >= 0 && i < K_COUNT) ? kKernNames[i] : ""; }

int lfds_kernel_times(lfds_plan* P, double* ms, int* launches) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  int rc;
  if ((rc = prof_drain(P))) return rc;
  for (int i = 0; i < K_COUNT; ++i) {
    if (ms) ms[i] = P->prof.ms[ST_COUNT + i];
    if (launches) launches[i] = P->prof.launches[ST_COUNT + i];
    P->prof.ms[ST_COUNT + i] = 0;
    P->prof.launches[ST_COUNT + i] = 0;
  }
  return LFDS_OK;
}

const char* lfds_last_error(void) { return g_err.c_str(); }
const char* lfds_version(void) { return "lfds 0.1 (sm_100a)"; }

// min over (l, m, t) of |lambda_l + mu_m + theta_t| for every block (steps 2, 6) and the global
// family (step 5) on the device (lfds_margin.cu); LFDS_ERESONANCE below opt.resonance_tol
static int resonance_margins(lfds_plan* P, const std::vector<zc>& za, const std::vector<zc>& zg,
                             const std::vector<zc>& zcv, const std::vector<zc>& ze) {
  std::vector<zc> theta;
  std::string err;
  if (!z_pencil_values(za, zg, zcv, ze, theta, err)) return fail(LFDS_EEIG, "z pencil: %s", err.c_str());
  std::stable_sort(theta.begin(), theta.end(), [](const zc& a, const zc& b) {
    return a.real() < b.real() || (a.real() == b.real() && a.imag() < b.imag());
  });
  const Axis& X = P->ax[0];
  const Axis& Y = P->ax[1];
  std::vector<zc> ev;
  std::vector<MarginSet> sets;
  auto put = [&](const std::vector<zc>& v) { int64_t o = (int64_t)ev.size(); ev.insert(ev.end(), v.begin(), v.end()); return o; };
  std::vector<int64_t> bxo, byo;
  for (auto& b : X.blocks) bxo.push_back(put(b.B.lam));
  for (auto& b : Y.blocks) byo.push_back(put(b.B.lam));
  for (int j = 0; j < P->nby; ++j)
    for (int i = 0; i < P->nbx; ++i) sets.push_back({bxo[i], byo[j], X.blocks[i].n, Y.blocks[j].n});
  const bool glob = X.G.n > 0 && Y.G.n > 0;
  if (glob) sets.push_back({put(X.G.lam), put(Y.G.lam), X.G.n, Y.G.n});
  const int nz = P->nz, ns = (int)sets.size();
  (void)cudaGetLastError();  // (stale non-sticky errors of the caller)
  double2 *d_ev = nullptr, *d_th = nullptr;
  MarginSet* d_sets = nullptr;
  unsigned long long* d_out = nullptr;
  std::vector<double2> hev(ev.size()), hth(nz);
  for (size_t q = 0; q < ev.size(); ++q) hev[q] = make_double2(ev[q].real(), ev[q].imag());
  for (int t = 0; t < nz; ++t) hth[t] = make_double2(theta[t].real(), theta[t].imag());
  std::vector<unsigned long long> keys(ns);
  cudaError_t e = cudaMalloc(&d_ev, hev.size() * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&d_th, hth.size() * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&d_sets, ns * sizeof(MarginSet));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, ns * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpy(d_ev, hev.data(), hev.size() * sizeof(double2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_th, hth.data(), hth.size() * sizeof(double2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_sets, sets.data(), ns * sizeof(MarginSet), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_margins(d_ev, d_sets, ns, d_th, nz, d_out, 0);
  if (e == cudaSuccess) e = cudaMemcpy(keys.data(), d_out, ns * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d_ev); cudaFree(d_th); cudaFree(d_sets); cudaFree(d_out);
  CUDA_TRY(e);
  double tmax = 0;
  for (auto& t : theta) tmax = std::max(tmax, std::abs(t));
  auto amax = [](const std::vector<zc>& v, int64_t o, int n) {
    double m = 0;
    for (int q = 0; q < n; ++q) m = std::max(m, std::abs(v[o + q]));
    return m;
  };
  lfds_info& I = P->info;
  for (int s = 0; s < ns; ++s) {
    const MarginSet& S = sets[s];
    const uint32_t idx = (uint32_t)(keys[s] & 0xffffffffull);
    const int l = (int)(idx % (uint32_t)S.nx), m = (int)((idx / (uint32_t)S.nx) % (uint32_t)S.ny),
              t = (int)(idx / ((uint32_t)S.nx * (uint32_t)S.ny));
    const double mg = std::abs(ev[S.lx + l] + ev[S.ly + m] + theta[t]);  // exact value at the argmin
    const double rel = mg / (amax(ev, S.lx, S.nx) + amax(ev, S.ly, S.ny) + tmax);
    if (glob && s == ns - 1) {
      I.margin_global = mg; I.margin_global_rel = rel;
      I.margin_global_lmt[0] = l; I.margin_global_lmt[1] = m; I.margin_global_lmt[2] = t;
    } else if (I.margin_block_rel < 0 || rel < I.margin_block_rel) {
      I.margin_block = mg; I.margin_block_rel = rel;
      I.margin_block_ij[0] = s % P->nbx; I.margin_block_ij[1] = s / P->nbx;
      I.margin_block_lmt[0] = l; I.margin_block_lmt[1] = m; I.margin_block_lmt[2] = t;
    }
  }
  if (!glob) {  // a single block is the global problem
    I.margin_global = I.margin_block; I.margin_global_rel = I.margin_block_rel;
    for (int q = 0; q < 3; ++q) I.margin_global_lmt[q] = I.margin_block_lmt[q];
  }
  const double tol = P->opt.resonance_tol;
  if (tol > 0 && glob && I.margin_global_rel < tol)
    return fail(LFDS_ERESONANCE, "resonance: global z-systems singular to %.3g (relative margin %.3g < %.3g) at "
                "harmonic (l, m) = (%d, %d), z-mode t = %d", I.margin_global, I.margin_global_rel, tol,
                I.margin_global_lmt[0], I.margin_global_lmt[1], I.margin_global_lmt[2]);
  if (tol > 0 && I.margin_block_rel < tol)
    return fail(LFDS_ERESONANCE, "resonance: block (%d, %d) z-systems singular to %.3g (relative margin %.3g < %.3g) "
                "at harmonic (l, m) = (%d, %d), z-mode t = %d", I.margin_block_ij[0], I.margin_block_ij[1],
                I.margin_block, I.margin_block_rel, tol, I.margin_block_lmt[0], I.margin_block_lmt[1],
                I.margin_block_lmt[2]);
  return LFDS_OK;
}

static int setup_axis(Axis& A, int N, const lfds_z* h, int nif, const int* iface, bool need_global, const char* name) {
  A.N = N;
  A.h.resize(N + 1);
  for (int t = 0; t <= N; ++t) {
    A.h[t] = zc(h[t].re, h[t].im);
    if (!(A.h[t].real() > 0)) return fail(LFDS_EINVAL, "%s: step h_%d has Re(h) <= 0", name, t);
  }
  A.hh.resize(N);
  for (int i = 0; i < N; ++i) A.hh[i] = 0.5 * (A.h[i] + A.h[i + 1]);
  A.iface.assign(iface, iface + nif);
  // step 5 contracts over the interface planes on the tensor pipe with |I| padded to 8, 16 or 32
  // (32: z-modal form only, checked once the z tables are known)
  if (nif > 32) return fail(LFDS_EINVAL, "%s: at most 32 interfaces (33 blocks) per axis, got %d", name, nif);
  for (int a = 0; a < nif; ++a) {
    int v = A.iface[a];
    if (v < 2 || v > N - 1) return fail(LFDS_EINVAL, "%s: interface node %d outside 2..N-1", name, v);
    if (a > 0 && v < A.iface[a - 1] + 2) return fail(LFDS_EINVAL, "%s: interfaces must be sorted and >= 2 apart", name);
  }
  A.blk_of.assign(N, -1);
  std::vector<int> cuts;
  cuts.push_back(0);
  for (int v : A.iface) cuts.push_back(v);
  cuts.push_back(N + 1);
  for (size_t c = 0; c + 1 < cuts.size(); ++c) {
    AxisBlock b;
    b.lo = cuts[c] + 1;
    b.n = cuts[c + 1] - 1 - cuts[c];
    for (int p = 0; p < b.n; ++p) A.blk_of[b.lo - 1 + p] = (int)A.blocks.size();
    A.blocks.push_back(b);
  }
  std::string err;
  for (auto& b : A.blocks) {
    std::vector<zc> hs(A.h.begin() + (b.lo - 1), A.h.begin() + (b.lo + b.n));
    if (!pencil_basis(hs, b.B, err)) return fail(LFDS_EEIG, "%s block at node %d: %s", name, b.lo, err.c_str());
  }
  if (need_global) {
    if (!pencil_basis(A.h, A.G, err)) return fail(LFDS_EEIG, "%s global basis: %s", name, err.c_str());
  }
  return LFDS_OK;
}

int lfds_setup_grid(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                    const lfds_z* sigma_node, const lfds_z* sigma_edge, lfds_z lambda, int n_if_x, const int* if_x,
                    int n_if_y, const int* if_y, const lfds_options* opt, lfds_plan** out) {
  auto t0 = std::chrono::steady_clock::now();
  if (!out) return fail(LFDS_EINVAL, "out is NULL");
  *out = nullptr;
  if (nx < 1 || ny < 1 || nz < 1) return fail(LFDS_EINVAL, "sizes must be >= 1 (nx=%d ny=%d nz=%d)", nx, ny, nz);
  if (nz > 512) return fail(LFDS_EINVAL, "nz=%d > 512 is not supported by the warp z-solver", nz);
  if (!hx || !hy || !hz || !sigma_node || !sigma_edge) return fail(LFDS_EINVAL, "NULL input array");
  if ((n_if_x && !if_x) || (n_if_y && !if_y) || n_if_x < 0 || n_if_y < 0) return fail(LFDS_EINVAL, "bad interface arrays");
  std::unique_ptr<lfds_plan> P(new lfds_plan());
  if (opt) P->opt = *opt;
  else lfds_default_options(&P->opt);
  if (P->opt.refine < -1 || P->opt.refine > 8) return fail(LFDS_EINVAL, "refine must be -1..8");
  int rc;
  const bool need_global = n_if_x + n_if_y > 0;
  if ((rc = setup_axis(P->ax[0], nx, hx, n_if_x, if_x, need_global, "x"))) return rc;
  if ((rc = setup_axis(P->ax[1], ny, hy, n_if_y, if_y, need_global, "y"))) return rc;
  P->nz = nz;
  P->hz.resize(nz + 1);
  P->sig_edge.resize(nz + 1);
  P->sig_node.resize(nz);
  for (int k = 0; k <= nz; ++k) {
    P->hz[k] = zc(hz[k].re, hz[k].im);
    P->sig_edge[k] = zc(sigma_edge[k].re, sigma_edge[k].im);
    if (!(P->hz[k].real() > 0)) return fail(LFDS_EINVAL, "z: step h_%d has Re(h) <= 0", k);
    if (!(P->sig_edge[k].real() > 0)) return fail(LFDS_EINVAL, "sigma_edge[%d] has Re <= 0", k);
  }
  for (int k = 0; k < nz; ++k) {
    P->sig_node[k] = zc(sigma_node[k].re, sigma_node[k].im);
    if (!(P->sig_node[k].real() > 0)) return fail(LFDS_EINVAL, "sigma_node[%d] has Re <= 0", k);
  }
  P->lam = zc(lambda.re, lambda.im);
  P->hhz.resize(nz);
  for (int k = 0; k < nz; ++k) P->hhz[k] = 0.5 * (P->hz[k] + P->hz[k + 1]);
  if (P->opt.dtype == LFDS_F64) {
    bool ok = P->lam.imag() == 0;
    for (auto& a : P->ax)
      for (auto& z : a.h) ok = ok && z.imag() == 0;
    for (auto& z : P->hz) ok = ok && z.imag() == 0;
    for (auto& z : P->sig_edge) ok = ok && z.imag() == 0;
    for (auto& z : P->sig_node) ok = ok && z.imag() == 0;
    if (!ok) return fail(LFDS_EINVAL, "LFDS_F64 requires real steps, sigma and lambda");
  }
  Axis& X = P->ax[0];
  Axis& Y = P->ax[1];
  P->nbx = (int)X.blocks.size();
  P->nby = (int)Y.blocks.size();
  P->mpad = 0;
  P->lpad = 0;
  for (auto& b : Y.blocks) P->mpad = std::max(P->mpad, b.n);
  for (auto& b : X.blocks) P->lpad = std::max(P->lpad, b.n);
  P->fpad = std::max(P->mpad, P->lpad);
  // eigen diagnostics
  double mres = 0, mbio = 0;
  for (auto& a : P->ax) {
    for (auto& b : a.blocks) { mres = std::max(mres, b.B.residual); mbio = std::max(mbio, b.B.biorth); }
    if (a.G.n) { mres = std::max(mres, a.G.residual); mbio = std::max(mbio, a.G.biorth); }
  }
  if (!(mres < 1e-8) || !(mbio < 1e-3))
    return fail(LFDS_EEIG, "eigenbasis check failed: residual %.3e, biorthonormality %.3e", mres, mbio);
  // ---- device tables
  TabBuilder T;
  for (auto& a : P->ax) {
    for (auto& b : a.blocks) {
      const int n = b.n;
      std::vector<zc> F((size_t)n * n);
      for (int l = 0; l < n; ++l)
        for (int p = 0; p < n; ++p) F[(size_t)l * n + p] = b.B.W[(size_t)p * n + l] * a.hh[b.lo - 1 + p];
      b.F = T.put(F);
      b.W = T.put(b.B.W);
      b.lam = T.put(b.B.lam);
      if (b.B.kind == 0 && dst_supported(b.n)) {
        const double h = a.h[b.lo - 1].real(), Nn = b.n + 1.0;
        b.dst = true;
        b.dst_fwd = std::sqrt(2.0 * h / Nn);
        b.dst_inv = std::sqrt(2.0 / (h * Nn));
      }
      if (b.B.kind != 2) {
        bool real = true;
        for (auto& z : F) real = real && z.imag() == 0;
        if (real) {
          b.Fr = T.put_real(F);
          b.Wr = T.put_real(b.B.W);
        }
      }
    }
    if (a.G.n) {
      const int N = a.N;
      std::vector<int> perm(N);
      std::iota(perm.begin(), perm.end(), 0);
      bool palin = N >= 2;
      for (int t = 0; t <= N && palin; ++t) palin = a.h[t] == a.h[N - t];
      a.gpal = false;
      a.ne = 0;
      if (palin) {  // classify every column by its exact mirror symmetry
        std::vector<int> ev, od;
        bool ok = true;
        for (int c = 0; c < N && ok; ++c) {
          int pm = 0;
          for (int p = 1; p < N / 2; ++p)
            if (std::abs(a.G.W[(size_t)p * N + c]) > std::abs(a.G.W[(size_t)pm * N + c])) pm = p;
          const zc w = a.G.W[(size_t)pm * N + c], wm = a.G.W[(size_t)(N - 1 - pm) * N + c];
          if (w == zc(0)) ok = false;
          else if (wm == w) ev.push_back(c);
          else if (wm == -w) od.push_back(c);
          else ok = false;
        }
        if (ok && (int)ev.size() == (N + 1) / 2) {
          for (int c = 0; c < (int)ev.size(); ++c) perm[c] = ev[c];
          for (int c = 0; c < (int)od.size(); ++c) perm[ev.size() + c] = od[c];
          a.gpal = true;
          a.ne = (int)ev.size();
        }
      }
      std::vector<zc> Wp((size_t)N * N), lp(N);
      for (int p = 0; p < N; ++p)
        for (int c = 0; c < N; ++c) Wp[(size_t)p * N + c] = a.G.W[(size_t)p * N + perm[c]];
      for (int c = 0; c < N; ++c) lp[c] = a.G.lam[perm[c]];
      a.Wg = T.put(Wp);
      a.lamg = T.put(lp);
      std::vector<zc> WI((size_t)a.iface.size() * N);
      for (size_t q = 0; q < a.iface.size(); ++q)
        for (int l = 0; l < N; ++l) WI[q * N + l] = Wp[(size_t)(a.iface[q] - 1) * N + l];
      a.WI = T.put(WI);
    }
    a.hoff = T.put(a.h);
    a.hhoff = T.put(a.hh);
  }
  // z tables: T(s) row k = a_k x_{k-1} + (g_k + s e_k) x_k + c_k x_{k+1}
  std::vector<zc> za(nz), zg(nz), zcv(nz), ze(nz), sa(nz), sg(nz), scv(nz), se(nz);
  for (int k = 0; k < nz; ++k) {
    zc lo = P->sig_edge[k] / P->hz[k], hi = P->sig_edge[k + 1] / P->hz[k + 1];
    za[k] = k > 0 ? lo : zc(0);
    zcv[k] = k + 1 < nz ? hi : zc(0);
    zg[k] = -(lo + hi) + P->lam * P->hhz[k];
    ze[k] = P->sig_node[k] * P->hhz[k];
    sa[k] = za[k] / P->hhz[k];
    scv[k] = zcv[k] / P->hhz[k];
    sg[k] = zg[k] / P->hhz[k];
    se[k] = P->sig_node[k];
    for (auto* z : {&za[k], &zg[k], &zcv[k], &ze[k]})
      if (z->imag() != 0) P->real_z = false;
  }
  P->zt_plain = ZTab{T.put(za), T.put(zg), T.put(zcv), T.put(ze)};
  if (P->opt.s5_modal && P->real_z && (!X.iface.empty() || !Y.iface.empty())) {
    // z modal basis of the step-5 systems T(s) = A' + s E (A' = tridiag(za, zg, zcv), E = diag(ze))
    std::vector<double> a(nz), g(nz), c(nz), e(nz), theta, Z;
    for (int k = 0; k < nz; ++k) { a[k] = za[k].real(); g[k] = zg[k].real(); c[k] = zcv[k].real(); e[k] = ze[k].real(); }
    double zres = 0, zorth = 0;
    std::string zerr;
    if (!z_modal_basis(a, g, c, e, theta, Z, zres, zorth, zerr))
      return fail(LFDS_EEIG, "z modal basis: %s", zerr.c_str());
    if (!(zres < 1e-12) || !(zorth < 1e-12))
      return fail(LFDS_EEIG, "z modal basis: residual %.3g, orthonormality %.3g", zres, zorth);
    std::vector<zc> zt((size_t)nz * nz), zf((size_t)nz * nz), th(nz);
    for (int k = 0; k < nz; ++k)
      for (int t = 0; t < nz; ++t) {
        zf[(size_t)k * nz + t] = Z[(size_t)k * nz + t];
        zt[(size_t)t * nz + k] = Z[(size_t)k * nz + t];
      }
    for (int t = 0; t < nz; ++t) th[t] = theta[t];
    P->t_zt = T.put_real(zt);
    P->t_zf = T.put_real(zf);
    P->t_theta = T.put(th);
    P->s5m = true;
    P->info.z_eig_residual = zres;
    P->info.z_eig_orth = zorth;
  }
  P->zt_scaled = ZTab{T.put(sa), T.put(sg), T.put(scv), T.put(se)};
  if (!P->s5m && std::max(X.iface.size(), Y.iface.size()) > 16)
    return fail(LFDS_EINVAL, "more than 16 interfaces per axis need the z-modal step 5 (real z tables, "
                             "options.s5_modal = 1)");
  {  // step-6 lifting RHS is -sigma_k (sum of face terms): fold -sigma_k into the rows
    std::vector<zc> la(nz), lg(nz), lc(nz), le(nz);
    for (int k = 0; k < nz; ++k) {
      const zc f = -1.0 / P->sig_node[k];
      la[k] = sa[k] * f; lg[k] = sg[k] * f; lc[k] = scv[k] * f; le[k] = se[k] * f;
    }
    P->zt_lift = ZTab{T.put(la), T.put(lg), T.put(lc), T.put(le)};
  }
  for (auto& a : P->ax)  // FFT twiddles W_L^j = exp(-2 pi i j/L) for the sine transforms in use
    for (auto& b : a.blocks) {
    const int L = 2 * (b.n + 1);
    if (!b.dst || P->t_tw.count(L)) continue;
    std::vector<zc> tw(L);
    for (int j = 0; j < L; ++j) {
      const long double ang = -2.0L * 3.141592653589793238462643383279502884L * j / L;
      tw[j] = zc((double)std::cos(ang), (double)std::sin(ang));
    }
    P->t_tw[L] = T.put(tw);
  }
  {  // double-double stencil coefficients per node (long double, split into hi + lo):
     // x, y: cl_i = 1/(h_{i-1} hh_i), cr_i = 1/(h_i hh_i); z: sigma_{k-1/2}/(h_{k-1} hh_k), sigma_{k+1/2}/(h_k hh_k)
    using lc = std::complex<long double>;
    auto split_put = [&](const std::vector<lc>& v) {
      std::vector<zc> w(2 * v.size());
      for (size_t t = 0; t < v.size(); ++t) {
        const long double re = v[t].real(), im = v[t].imag();
        const double rh = (double)re, ih = (double)im;
        w[2 * t] = zc(rh, (double)(re - rh));
        w[2 * t + 1] = zc(ih, (double)(im - ih));
      }
      return T.put(w);
    };
    auto node_tab = [&](const std::vector<zc>& h, const std::vector<zc>* se) {
      const int n = (int)h.size() - 1;
      std::vector<lc> v(2 * n);
      for (int i = 0; i < n; ++i) {
        const lc h0(h[i]), h1(h[i + 1]), hh = (h0 + h1) / 2.0L;
        const lc s0 = se ? lc((*se)[i]) : lc(1), s1 = se ? lc((*se)[i + 1]) : lc(1);
        v[2 * i] = s0 / (h0 * hh);
        v[2 * i + 1] = s1 / (h1 * hh);
      }
      return split_put(v);
    };
    P->t_dd[0] = node_tab(P->ax[0].h, nullptr);
    P->t_dd[1] = node_tab(P->ax[1].h, nullptr);
    P->t_dd[2] = node_tab(P->hz, &P->sig_edge);
  }
  P->t_hz = T.put(P->hz);
  P->t_hhz = T.put(P->hhz);
  P->t_sig = T.put(P->sig_node);
  P->t_sige = T.put(P->sig_edge);
  P->t_ifx = T.put_ints(X.iface);
  P->t_ify = T.put_ints(Y.iface);
  P->t_bx = T.put_ints(X.blk_of);
  P->t_by = T.put_ints(Y.blk_of);
  std::vector<int> xlo, ylo;
  for (auto& b : X.blocks) xlo.push_back(b.lo);
  for (auto& b : Y.blocks) ylo.push_back(b.lo);
  P->t_xlo = T.put_ints(xlo);
  P->t_ylo = T.put_ints(ylo);
  P->tab_elems = T.v.size();
  if (P->opt.device >= 0) {
    CUDA_TRY(cudaSetDevice(P->opt.device));
    CUDA_TRY(cudaMalloc(&P->d_tab, T.v.size() * sizeof(double2)));
    CUDA_TRY(cudaMemcpy(P->d_tab, T.v.data(), T.v.size() * sizeof(double2), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMallocHost(&P->h_piv, sizeof(double)));
    *P->h_piv = -1.0;
  }
  // ---- resonance margins of the block and global z-systems (reading R13; never regularised)
  {
    lfds_info& I = P->info;
    I.margin_global = I.margin_global_rel = I.margin_block = I.margin_block_rel = -1.0;
    for (int q = 0; q < 3; ++q) I.margin_global_lmt[q] = I.margin_block_lmt[q] = -1;
    I.margin_block_ij[0] = I.margin_block_ij[1] = -1;
    if (P->opt.device >= 0 && (int64_t)nx * ny * nz < (int64_t)UINT32_MAX) {
      if ((rc = resonance_margins(P.get(), za, zg, zcv, ze))) {
        const std::string msg = g_err;
        lfds_destroy(P.release());  // device tables already allocated
        g_err = msg;
        return rc;
      }
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  lfds_info& I = P->info;
  I.nx = nx; I.ny = ny; I.nz = nz; I.nbx = P->nbx; I.nby = P->nby; I.n_if_x = n_if_x; I.n_if_y = n_if_y;
  I.real_z = P->real_z ? 1 : 0;
  I.setup_seconds = std::chrono::duration<double>(t1 - t0).count();
  I.eig_max_residual = mres;
  I.eig_max_biorth = mbio;
  I.device_table_bytes = T.v.size() * sizeof(double2);
  I.s5_modal = P->s5m ? 1 : 0;
  I.global_fold = (X.gpal ? 1 : 0) | (Y.gpal ? 2 : 0);
  I.n_plane_dst = 0;  // the fused2() rule of build_pass (complex data only)
  if (P->opt.plane_dst && P->opt.dtype != LFDS_F64)
    for (auto& by : Y.blocks)
      for (auto& bx : X.blocks) I.n_plane_dst += bx.dst && by.dst && bx.n == by.n && dst2_supported(bx.n);
  // the xplane() rule of build_pass (complex data only).  The plane form pays when the blocks it
  // applies to carry the solve (C5: every block); a few small corner blocks among sine or large
  // blocks (C3, C2, C4q, C4j) only add launches to launch-bound steps (C3 1.32 -> 1.41 ms), so it
  // is used when those blocks hold at least half of the block unknowns.
  I.n_plane_dense = 0;
  if (xplane_on() && P->opt.dtype != LFDS_F64) {
    int64_t el_x = 0, el_all = 0;
    int cnt = 0;
    for (auto& by : Y.blocks)
      for (auto& bx : X.blocks) {
        const bool f2 = P->opt.plane_dst && bx.dst && by.dst && bx.n == by.n && dst2_supported(bx.n);
        const bool xp = !f2 && !bx.dst && !by.dst && bx.n <= 32 && by.n <= 32;
        el_all += (int64_t)bx.n * by.n;
        if (xp) { el_x += (int64_t)bx.n * by.n; ++cnt; }
      }
    P->xplane_ok = 2 * el_x >= el_all && cnt > 0;
    if (P->xplane_ok) I.n_plane_dense = cnt;
  }
  *out = P.release();
  return LFDS_OK;
}

static int chunk_of(const lfds_plan* P, int nrhs) {
  int c = P->opt.rhs_chunk > 0 ? P->opt.rhs_chunk : nrhs;
  return std::max(1, std::min(c, nrhs));
}

size_t lfds_workspace_bytes(const lfds_plan* cp, int nrhs) {
  lfds_plan* P = const_cast<lfds_plan*>(cp);
  if (!P || nrhs < 1 || !P->d_tab) return 0;
  int R = chunk_of(P, nrhs);
  int in_real = P->opt.dtype == LFDS_F64;
  PassPlan* pp;
  if (get_pass(P, R, in_real, in_real, &pp)) return 0;
  size_t total = pp->total;
  // refinement passes run the complex pass plan (its own layout in the same workspace; for a
  // complex plan it is the main one); a last chunk smaller than R has a smaller layout
  if (P->opt.refine != 0) {
    if (get_pass(P, R, 0, 0, &pp)) return 0;
    total = std::max(total, pp->total);
  }
  return total;
}

size_t lfds_workspace_bytes_host(const lfds_plan* P, int nrhs) {
  size_t ws = lfds_workspace_bytes(P, nrhs);
  if (!ws) return 0;
  size_t el = P->opt.dtype == LFDS_F64 ? 8 : 16;
  size_t vol = (size_t)P->ax[0].N * P->ax[1].N * P->nz * nrhs * el;
  return ws + 2 * al256(vol);
}

static int solve_impl(lfds_plan* P, const void* f_dev, void* u_dev, int nrhs, void* ws, size_t ws_bytes, cudaStream_t st) {
  (void)cudaGetLastError();  // a stale non-sticky error of the caller is not ours to report
  // a partitioned plan computes only its own blocks: whole solves must go through the phases
  if (P->sharded) return fail(LFDS_EINVAL, "partitioned plan: use lfds_solve_phase with the two exchanges");
  const int R = chunk_of(P, nrhs);
  const int dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
  const size_t el = dt ? 8 : 16;
  const int64_t vol = (int64_t)P->ax[0].N * P->ax[1].N * P->nz;
  P->launches = 0;
  P->report = lfds_report{};
  P->report.min_pivot_ratio = 1.0;
  // the pivot monitor lives at offset 0 of the workspace in every pass plan (RED first): one
  // fill per solve, every chunk and refinement pass takes its min into the same word
  double* red0 = reinterpret_cast<double*>(ws);
  CUDA_TRY(launch_fill_minpiv(red0, st));
  double maxres[9] = {0};
  int passes_done = 0;
  for (int r0 = 0; r0 < nrhs; r0 += R) {
    const int Rc = std::min(R, nrhs - r0);
    PassPlan *pp_main, *pp_ref = nullptr;
    int rc;
    if ((rc = get_pass(P, Rc, dt, dt, &pp_main))) return rc;
    if (P->opt.refine != 0 && (rc = get_pass(P, Rc, 0, 0, &pp_ref))) return rc;
    const size_t need = std::max(pp_main->total, pp_ref ? pp_ref->total : size_t(0));
    if (ws_bytes < need) return fail(LFDS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
    char* w = reinterpret_cast<char*>(ws);
    Bufs b{};
    b.p[B_TAB] = P->d_tab;
    b.p[B_F] = const_cast<char*>(reinterpret_cast<const char*>(f_dev)) + (size_t)r0 * vol * el;
    b.p[B_U] = reinterpret_cast<char*>(u_dev) + (size_t)r0 * vol * el;
    b.p[B_MS] = w + pp_main->off_ms;
    b.p[B_T1] = w + pp_main->off_t1;
    b.p[B_IF] = w + pp_main->off_if;
    b.p[B_RED] = w + pp_main->off_red;
    b.p[B_CK] = w + pp_main->off_ck;
    double* red = reinterpret_cast<double*>(b.p[B_RED]);
    if ((rc = run_pass(P, *pp_main, b, Rc, dt, dt, st))) return rc;
    int passes = 1;
    if (P->opt.refine != 0) {
      // the refinement pass runs pp_ref on pp_ref's own layout of the workspace (an f64 plan's
      // real main pass has another); the residual lives past all of pp_ref's buffers
      double2* res = reinterpret_cast<double2*>(w + pp_ref->off_res);
      double* norms = red + 8;
      const Axis& X = P->ax[0];
      const Axis& Y = P->ax[1];
      double prev = 1e300;
      const int maxref = P->opt.refine < 0 ? 8 : P->opt.refine;
      for (int it = 0; it <= maxref; ++it) {
        // a fixed pass count needs no residual after the last correction (auto mode does: it
        // decides whether to continue from it)
        if (it == maxref && P->opt.refine > 0) break;
        // auto mode reads the residual norms back (it decides on them, which synchronises the
        // stream); a fixed pass count stays asynchronous
        const bool auto_mode = P->opt.refine < 0;
        if (auto_mode) CUDA_TRY(cudaMemsetAsync(norms, 0, sizeof(double) * 2 * Rc, st));
        cudaEvent_t ra = nullptr, ra2 = nullptr, rb2k = nullptr;  // stage and kernel-kind events
        if (P->opt.profile) { ra = P->prof.get(); prof_record(ra, st); }
        if (P->opt.profile >= 2) { ra2 = P->prof.get(); prof_record(ra2, st); }
        CUDA_TRY(launch_residual(X.N, Y.N, P->nz, Rc, dt, P->opt.residual_dd, 1, X.hoff, Y.hoff, P->t_hz, X.hhoff,
                                 Y.hhoff, P->t_hhz, P->t_sig, P->t_sige, make_double2(P->lam.real(), P->lam.imag()),
                                 P->t_dd, b.p[B_U], b.p[B_F], res, 1, auto_mode ? norms : nullptr, b, st));
        P->launches++;
        if (P->opt.profile >= 2) {
          rb2k = P->prof.get();
          prof_record(rb2k, st);
          P->prof.recs.push_back({ST_COUNT + K_RESID, 1, ra2, rb2k});
        }
        if (P->opt.profile) {
          cudaEvent_t rb2 = P->prof.get();
          prof_record(rb2, st);
          P->prof.recs.push_back({ST_RESID, 1, ra, rb2});
        }
        double worst = -1.0;
        if (auto_mode) {
          std::vector<double> hn(2 * Rc);
          CUDA_TRY(cudaMemcpyAsync(hn.data(), norms, sizeof(double) * 2 * Rc, cudaMemcpyDeviceToHost, st));
          CUDA_TRY(cudaStreamSynchronize(st));
          worst = 0;
          for (int r = 0; r < Rc; ++r) worst = std::max(worst, hn[2 * r + 1] > 0 ? std::sqrt(hn[2 * r] / hn[2 * r + 1]) : 0.0);
        }
        if (it < 9) maxres[it] = std::max(maxres[it], worst);
        if (it == maxref) break;
        if (P->opt.refine < 0 && (worst <= P->opt.refine_tol || worst > 0.5 * prev)) break;
        prev = worst;
        Bufs rb = b;
        rb.p[B_F] = res;
        rb.p[B_U] = res;
        rb.p[B_MS] = w + pp_ref->off_ms;
        rb.p[B_T1] = w + pp_ref->off_t1;
        rb.p[B_IF] = w + pp_ref->off_if;
        rb.p[B_RED] = w + pp_ref->off_red;  // == pp_main->off_red (RED first in every layout)
        rb.p[B_CK] = w + pp_ref->off_ck;
        if ((rc = run_pass(P, *pp_ref, rb, Rc, 0, 0, st))) return rc;
        cudaEvent_t xa = nullptr, xa2 = nullptr, xb2 = nullptr;
        if (P->opt.profile) { xa = P->prof.get(); prof_record(xa, st); }
        if (P->opt.profile >= 2) { xa2 = P->prof.get(); prof_record(xa2, st); }
        CUDA_TRY(launch_axpy_u(vol * Rc, dt, res, b.p[B_U], st));
        P->launches++;
        if (P->opt.profile >= 2) {
          xb2 = P->prof.get();
          prof_record(xb2, st);
          P->prof.recs.push_back({ST_COUNT + K_AXPY, 1, xa2, xb2});
        }
        if (P->opt.profile) {
          cudaEvent_t xb = P->prof.get();
          prof_record(xb, st);
          P->prof.recs.push_back({ST_AXPY, 1, xa, xb});
        }
        passes++;
      }
    }
    passes_done = std::max(passes_done, passes);
  }
  // stream-ordered copy of the monitor into pinned host memory (a graph node when captured):
  // lfds_get_report waits for it, the solve itself never synchronises for it
  CUDA_TRY(cudaMemcpyAsync(P->h_piv, red0, sizeof(double), cudaMemcpyDeviceToHost, st));
  P->piv_stream = st;
  P->piv_pending = true;
  P->report.passes = passes_done;
  for (int i = 0; i < 9; ++i) P->report.rel_residual[i] = maxres[i];
  P->report.n_kernel_launches = P->launches;
  return LFDS_OK;
}

// ------------------------------------------------------------------ heterogeneous media (GMRES)
size_t lfds_gmres_workspace_bytes(const lfds_plan* P, int restart) {
  if (!P || P->opt.device < 0 || restart < 1 || restart > 64) return 0;
  const size_t n = (size_t)P->ax[0].N * P->ax[1].N * P->nz;
  const size_t vec = al256(n * sizeof(double2));
  return vec * (size_t)(restart + 4) + al256((size_t)KRYLOV_DOT_BLOCKS * 80 * sizeof(double2)) +
         al256(80 * sizeof(double2)) + lfds_workspace_bytes(P, 1);
}

int lfds_gmres(lfds_plan* P, const void* dlam, const void* f, void* u, double tol, int maxit, int restart, void* ws,
               size_t ws_bytes, void* stream, lfds_krylov_report* rep) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (P->opt.device < 0) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (P->opt.dtype != LFDS_C128) return fail(LFDS_EINVAL, "lfds_gmres: complex128 plans only");
  if (restart < 1 || restart > 64 || maxit < 1 || !(tol > 0))
    return fail(LFDS_EINVAL, "lfds_gmres: need 1 <= restart <= 64, maxit >= 1, tol > 0");
  if (!dlam || !f || !u || !ws) return fail(LFDS_EINVAL, "lfds_gmres: NULL pointer");
  for (const void* q : {dlam, f, (const void*)u, (const void*)ws})
    if (reinterpret_cast<uintptr_t>(q) % 16) return fail(LFDS_EINVAL, "lfds_gmres: pointers must be 16-byte aligned");
  if (u == f || u == dlam) return fail(LFDS_EINVAL, "lfds_gmres: u must not alias f or dlam");
  const size_t need = lfds_gmres_workspace_bytes(P, restart);
  if (ws_bytes < need) return fail(LFDS_EINVAL, "lfds_gmres: workspace too small: %zu < %zu", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int m = restart;
  const int64_t n = (int64_t)P->ax[0].N * P->ax[1].N * P->nz;
  const size_t vec = al256((size_t)n * sizeof(double2));
  const int64_t vs = (int64_t)(vec / sizeof(double2));
  char* w0 = static_cast<char*>(ws);
  double2* V = reinterpret_cast<double2*>(w0);                        // m + 1 basis vectors
  double2* W = reinterpret_cast<double2*>(w0 + vec * (m + 1));
  double2* S = W + vs;
  double2* Y = S + vs;
  double2* part = reinterpret_cast<double2*>(w0 + vec * (m + 4));
  double2* coef = reinterpret_cast<double2*>(reinterpret_cast<char*>(part) +
                                             al256((size_t)KRYLOV_DOT_BLOCKS * 80 * sizeof(double2)));
  void* sws = reinterpret_cast<char*>(coef) + al256(80 * sizeof(double2));
  const size_t sws_bytes = lfds_workspace_bytes(P, 1);
  const double2* F = static_cast<const double2*>(f);
  const double2* DL = static_cast<const double2*>(dlam);
  std::vector<double2> hp((size_t)KRYLOV_DOT_BLOCKS * 80);
  int kl = 0;  // kernels launched (all fast solves and vector kernels)
  // out[i] = <V_i, x> for i < cnt (and out[cnt] = <x, x> if with_self)
  auto dots = [&](int cnt, const double2* Vb, const double2* x, std::vector<zc>& out, int with_self = 0) -> int {
    CUDA_TRY(launch_dots(n, cnt, Vb, vs, x, part, st, with_self));
    ++kl;
    CUDA_TRY(cudaMemcpyAsync(hp.data(), part, sizeof(double2) * hp.size(), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const int tot = cnt + (with_self ? 1 : 0);
    out.assign(tot, zc(0));
    for (int b = 0; b < KRYLOV_DOT_BLOCKS; ++b)  // fixed order: deterministic
      for (int i = 0; i < tot; ++i) out[i] += zc(hp[(size_t)b * 80 + i].x, hp[(size_t)b * 80 + i].y);
    return LFDS_OK;
  };
  auto axpy = [&](int cnt, const std::vector<zc>& c, double2* target) -> int {
    std::vector<double2> hc(cnt);
    for (int i = 0; i < cnt; ++i) hc[i] = make_double2(c[i].real(), c[i].imag());
    CUDA_TRY(cudaMemcpyAsync(coef, hc.data(), sizeof(double2) * cnt, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_maxpy(n, cnt, V, vs, coef, target, st));
    ++kl;
    CUDA_TRY(cudaStreamSynchronize(st));  // hc must outlive the copy
    return LFDS_OK;
  };
  // W += V c and ||W||^2 of the result in the same sweep (the Gram-Schmidt update)
  auto axpy_norm = [&](int cnt, const std::vector<zc>& c, double& nrm2) -> int {
    std::vector<double2> hc(cnt);
    for (int i = 0; i < cnt; ++i) hc[i] = make_double2(c[i].real(), c[i].imag());
    CUDA_TRY(cudaMemcpyAsync(coef, hc.data(), sizeof(double2) * cnt, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_maxpy_norm(n, cnt, V, vs, coef, W, part, st));
    ++kl;
    CUDA_TRY(cudaMemcpyAsync(hp.data(), part, sizeof(double2) * hp.size(), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    nrm2 = 0;
    for (int b = 0; b < KRYLOV_DOT_BLOCKS; ++b) nrm2 += hp[(size_t)b * 80].x;  // fixed order
    return LFDS_OK;
  };
  int rc;
  auto solve = [&](const void* src, void* dst) -> int {
    const int r = solve_impl(P, src, dst, 1, sws, sws_bytes, st);
    kl += P->launches;
    return r;
  };
  std::vector<zc> d;
  if ((rc = dots(1, F, F, d))) return rc;
  const double beta0 = std::sqrt(std::max(0.0, d[0].real()));
  if (rep) *rep = lfds_krylov_report{0, 0, 0.0};
  if (beta0 == 0) {
    CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(double2) * (size_t)n, st));
    return LFDS_OK;
  }
  CUDA_TRY(cudaMemsetAsync(Y, 0, sizeof(double2) * (size_t)n, st));
  CUDA_TRY(launch_scale(n, make_double2(1.0 / beta0, 0), F, V, st));
  double beta = beta0, res = 1.0;
  int it = 0, cycles = 0;
  bool conv = false, have_sy = false;
  std::vector<zc> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), h, h2;
  while (true) {
    std::fill(H.begin(), H.end(), zc(0));
    std::fill(g.begin(), g.end(), zc(0));
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      double2* Vj = V + (int64_t)j * vs;
      if ((rc = solve(Vj, S))) return rc;   // S V_j
      // (I + dlam S) V_j = V_j + z with z = dlam S V_j: orthogonalise z only (its V_j part is
      // exact: H[j][j] gets + 1), so no cancellation against the identity part of the operator
      CUDA_TRY(launch_fdie(n, nullptr, DL, S, W, st));                      // W = z = dlam S V_j
      ++kl;
      h.assign(j + 1, zc(0));
      double wn2 = 0, wn2_new = 0;
      for (int pass = 0; pass < 2; ++pass) {  // classical Gram-Schmidt, repeated when needed
        if ((rc = dots(j + 1, V, W, h2, pass == 0))) return rc;
        if (pass == 0) wn2 = h2[j + 1].real();
        std::vector<zc> c(j + 1);
        for (int i = 0; i <= j; ++i) { c[i] = -h2[i]; h[i] += h2[i]; }
        if ((rc = axpy_norm(j + 1, c, wn2_new))) return rc;
        // Kahan-Parlett: a second pass only if the projection removed most of w (||w'|| < ||w|| / sqrt2)
        if (wn2_new >= 0.5 * wn2) break;
        wn2 = wn2_new;
      }
      const double hn = std::sqrt(std::max(0.0, wn2_new));
      h[j] += 1.0;  // the identity part of (I + dlam S) V_j
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = h[i];
      for (int i = 0; i < j; ++i) {  // previous Givens rotations
        const zc a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * b;
        H[(size_t)(i + 1) * m + j] = -std::conj(sn[i]) * a + cs[i] * b;
      }
      const zc a = H[(size_t)j * m + j];
      if (std::abs(a) == 0) {
        cs[j] = 0;
        sn[j] = 1;
        H[(size_t)j * m + j] = hn;
      } else {
        const double t = std::hypot(std::abs(a), hn);
        const zc al = a / std::abs(a);
        cs[j] = std::abs(a) / t;
        sn[j] = al * hn / t;
        H[(size_t)j * m + j] = al * t;
      }
      g[j + 1] = -std::conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      ++it;
      jend = j + 1;
      res = std::abs(g[j + 1]) / beta0;
      const bool stop = res <= tol || it >= maxit || hn == 0;
      if (!stop && j + 1 < m) CUDA_TRY(launch_scale(n, make_double2(1.0 / hn, 0), W, V + (int64_t)(j + 1) * vs, st));
      if (stop) break;
    }
    std::vector<zc> c(jend);  // R c = g, y += V c
    for (int i = jend - 1; i >= 0; --i) {
      zc sacc = g[i];
      for (int k = i + 1; k < jend; ++k) sacc -= H[(size_t)i * m + k] * c[k];
      c[i] = sacc / H[(size_t)i * m + i];
    }
    if ((rc = axpy(jend, c, Y))) return rc;
    ++cycles;
    if (res <= tol) { conv = true; break; }
    if (it >= maxit) break;
    // restart from the true preconditioned residual r = f - (y + dlam S y)
    if ((rc = solve(Y, S))) return rc;
    CUDA_TRY(launch_fdie_res(n, F, Y, DL, S, W, st));
    if ((rc = dots(1, W, W, d))) return rc;
    beta = std::sqrt(std::max(0.0, d[0].real()));
    res = beta / beta0;
    if (res <= tol) { conv = true; have_sy = true; break; }
    CUDA_TRY(launch_scale(n, make_double2(1.0 / beta, 0), W, V, st));
  }
  if (have_sy) CUDA_TRY(cudaMemcpyAsync(u, S, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  else if ((rc = solve(Y, u))) return rc;    // u = S y
  CUDA_TRY(cudaStreamSynchronize(st));
  if (rep) *rep = lfds_krylov_report{it, cycles, res};
  P->report.n_kernel_launches = kl;
  if (!conv) return fail(LFDS_ENOTCONVERGED, "lfds_gmres: %d iterations, relative residual %.3g > %.3g", it, res, tol);
  return LFDS_OK;
}

int lfds_nccl_unique_id(unsigned char* id) {
  if (!id) return fail(LFDS_EINVAL, "id is NULL");
  NcclApi& A = nccl();
  if (!A.ok) return fail(LFDS_ENCCL, "NCCL not found (dlopen libnccl.so.2; LFDS_NCCL_LIB overrides)");
  NcclId u{};
  const int r = A.get_unique_id(&u);
  if (r) return fail(LFDS_ENCCL, "ncclGetUniqueId: %s", A.error_string(r));
  std::memcpy(id, u.internal, sizeof u.internal);
  return LFDS_OK;
}

int lfds_set_comm(lfds_plan* P, const unsigned char* id, int rank, int world) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  NcclApi& A = nccl();
  for (NcclComm* c : {&P->comm_m, &P->comm_l, &P->comm})
    if (*c) {
      if (A.ok) A.comm_destroy(*c);
      *c = nullptr;
    }
  drop_graph(P);  // a captured sharded graph holds the old communicator's collectives
  if (!id) return LFDS_OK;  // back to caller-driven exchanges
  if (world < 1 || rank < 0 || rank >= world) return fail(LFDS_EINVAL, "bad rank %d of %d", rank, world);
  if (!A.ok) return fail(LFDS_ENCCL, "NCCL not found (dlopen libnccl.so.2; LFDS_NCCL_LIB overrides)");
  CUDA_TRY(cudaSetDevice(P->opt.device));
  NcclId u{};
  std::memcpy(u.internal, id, sizeof u.internal);
  const int r = A.comm_init_rank(&P->comm, world, u, rank);
  if (r) { P->comm = nullptr; return fail(LFDS_ENCCL, "ncclCommInitRank: %s", A.error_string(r)); }
  P->comm_rank = rank;
  P->comm_world = world;
  return LFDS_OK;
}

int lfds_set_comm_groups(lfds_plan* P, int color_m, int color_l) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  NcclApi& A = nccl();
  if (!P->comm) return fail(LFDS_EINVAL, "lfds_set_comm_groups: call lfds_set_comm first");
  if (!A.comm_split) return fail(LFDS_ENCCL, "ncclCommSplit not available in the loaded NCCL");
  for (NcclComm* c : {&P->comm_m, &P->comm_l})
    if (*c) { A.comm_destroy(*c); *c = nullptr; }
  int r = A.comm_split(P->comm, color_m, P->comm_rank, &P->comm_m, nullptr);
  if (!r) r = A.comm_split(P->comm, color_l, P->comm_rank, &P->comm_l, nullptr);
  if (r) return fail(LFDS_ENCCL, "ncclCommSplit: %s", A.error_string(r));
  return LFDS_OK;
}

// the three phases with both exchanges summed over the communicator on the solve stream
// (stream-ordered: no host round trip between the phases, and the whole sharded solve can be
// captured in a CUDA graph); nrhs in one pass, no refinement (as lfds_solve_phase)
static int solve_sharded_nccl(lfds_plan* P, const void* f_dev, void* u_dev, int nrhs, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  NcclApi& A = nccl();
  int rc;
  auto exchange = [&](int which) -> int {
    size_t off = 0, n = 0;
    int e;
    if ((e = lfds_exchange_layout(P, nrhs, which, &off, &n))) return e;
    if (!n) return LFDS_OK;
    double* x = reinterpret_cast<double*>(static_cast<char*>(ws) + off);
    if (which == 3 && P->comm_m && P->comm_l) {
      // R1~ rows are shared by the ranks of a y-mode group, R2~ rows by an x-mode group: each
      // half summed over its own group only (the rows outside a group's range are zero there)
      PassPlan* pp;
      if ((e = get_pass(P, nrhs, 0, 0, &pp))) return e;
      const size_t n1 = (size_t)(pp->r2t - pp->r1t) * 2;
      int r = A.all_reduce(x, x, n1, NCCL_FLOAT64, NCCL_SUM, P->comm_m, st);
      if (!r) r = A.all_reduce(x + n1, x + n1, n - n1, NCCL_FLOAT64, NCCL_SUM, P->comm_l, st);
      if (r) return fail(LFDS_ENCCL, "ncclAllReduce (exchange 3): %s", A.error_string(r));
      return LFDS_OK;
    }
    const int r = A.all_reduce(x, x, n, NCCL_FLOAT64, NCCL_SUM, P->comm, st);
    if (r) return fail(LFDS_ENCCL, "ncclAllReduce (exchange %d): %s", which, A.error_string(r));
    return LFDS_OK;
  };
  // phases 1, 2 (= 2a + 2b), 3 with exchanges 1 and 2; with the formation split 2a, exchange 3
  // (the ranks' R1~ / R2~ rows), 2b
  // (phase, exchange after it): 1 -> 1, 2 -> 2, 3;  split: 1 -> 1, 4 -> 3, 5 -> 2, 3
  const bool split = P->fm0 >= 0;
  const int phases[4][2] = {{1, 1}, {split ? 4 : 2, split ? 3 : 2}, {split ? 5 : 3, split ? 2 : 0}, {3, 0}};
  for (int q = 0; q < (split ? 4 : 3); ++q) {
    if ((rc = lfds_solve_phase(P, phases[q][0], f_dev, u_dev, nrhs, ws, ws_bytes, st))) return rc;
    if (phases[q][1] && (rc = exchange(phases[q][1]))) return rc;
  }
  return LFDS_OK;
}

int lfds_set_partition(lfds_plan* P, const int* block_owned, int l_begin, int l_end, int rank0) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  const int nblk = P->nbx * P->nby, Nx = P->ax[0].N;
  if (!block_owned) {  // back to the whole problem on this device
    P->own.clear();
    P->sharded = false;
    P->l_begin = 0;
    P->l_end = -1;
    P->rank0 = 1;
    P->m_begin = 0;
    P->m_end = -1;
    P->fm0 = P->fm1 = P->fl0 = P->fl1 = -1;
  } else {
    if (l_begin < 0 || l_end < l_begin || l_end > Nx) return fail(LFDS_EINVAL, "bad x-mode range [%d, %d) of %d", l_begin, l_end, Nx);
    P->fm0 = P->fm1 = P->fl0 = P->fl1 = -1;
    P->own.assign(block_owned, block_owned + nblk);
    P->sharded = true;
    P->l_begin = l_begin;
    P->l_end = l_end;
    P->rank0 = rank0 ? 1 : 0;
    P->m_begin = 0;
    P->m_end = -1;
  }
  drop_graph(P);
  for (auto& kv : P->passes) {  // descriptors depend on the owned blocks: rebuild lazily
    free_pass(kv.second);
  }
  P->passes.clear();
  return LFDS_OK;
}

int lfds_set_mode_rows(lfds_plan* P, int m_begin, int m_end) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  const int Ny = P->ax[1].N;
  if (!P->sharded) return fail(LFDS_EINVAL, "lfds_set_mode_rows: call lfds_set_partition first");
  if (!P->s5m) return fail(LFDS_EINVAL, "lfds_set_mode_rows: step 5 runs as z-sweeps (complex z or s5_modal = 0)");
  if (m_begin < 0 || m_end < m_begin || m_end > Ny || (m_begin % 64 && m_begin != Ny) || (m_end % 64 && m_end != Ny))
    return fail(LFDS_EINVAL, "bad y-mode range [%d, %d) of %d (multiples of 64)", m_begin, m_end, Ny);
  P->m_begin = m_begin;
  P->m_end = m_end;
  drop_graph(P);
  for (auto& kv : P->passes) {  // descriptors depend on the range: rebuild lazily
    free_pass(kv.second);
  }
  P->passes.clear();
  return LFDS_OK;
}

}  // extern "C"

int lfds::plane_layout(lfds_plan* P, PlaneLayout* out) {
  PassPlan* pp;
  int rc;
  if ((rc = get_pass(P, 1, 0, 0, &pp))) return rc;
  out->rx = pp->rx;
  out->ry = pp->ry;
  out->wx = pp->wx;
  out->wy = pp->wy;
  out->off_if = pp->off_if;
  return LFDS_OK;
}

extern "C" {

int lfds_set_formation_rows(lfds_plan* P, int m_begin, int m_end, int l_begin, int l_end) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (m_begin < 0) {  // off
    P->fm0 = P->fm1 = P->fl0 = P->fl1 = -1;
  } else {
    if (!P->sharded || !P->s5m)
      return fail(LFDS_EINVAL, "lfds_set_formation_rows: needs a partitioned plan with the z-modal step 5");
    if (m_end < m_begin || m_end > P->ax[1].N || l_begin < 0 || l_end < l_begin || l_end > P->ax[0].N)
      return fail(LFDS_EINVAL, "bad formation rows [%d, %d) x [%d, %d)", m_begin, m_end, l_begin, l_end);
    P->fm0 = m_begin; P->fm1 = m_end; P->fl0 = l_begin; P->fl1 = l_end;
  }
  drop_graph(P);
  for (auto& kv : P->passes) free_pass(kv.second);
  P->passes.clear();
  return LFDS_OK;
}

int lfds_exchange_layout(const lfds_plan* cp, int nrhs, int which, size_t* byte_offset, size_t* n_doubles) {
  lfds_plan* P = const_cast<lfds_plan*>(cp);
  if (!P || which < 1 || which > 4 || !byte_offset || !n_doubles) return fail(LFDS_EINVAL, "bad arguments");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  const int R = chunk_of(P, nrhs);
  if (R != nrhs) return fail(LFDS_EINVAL, "sharded solves take all right-hand sides in one pass (rhs_chunk)");
  PassPlan* pp;
  int rc = get_pass(P, R, P->opt.dtype == LFDS_F64, P->opt.dtype == LFDS_F64, &pp);
  if (rc) return rc;
  if (which == 3 && !pp->s5m) { *byte_offset = pp->off_if; *n_doubles = 0; return LFDS_OK; }
  // [RX, RY] / [P1, P2] / [R1~, R2~] / [WX, WY] (w on the planes)
  const int64_t lo = which == 1 ? pp->rx : which == 2 ? pp->p1 : which == 3 ? pp->r1t : pp->wx;
  const int64_t hi = which == 1 ? pp->r1 : which == 2 ? pp->gp : which == 3 ? pp->p1t : pp->gf;
  *byte_offset = pp->off_if + (size_t)lo * 16;
  *n_doubles = (size_t)(hi - lo) * 2;
  return LFDS_OK;
}

int lfds_solve_phase(lfds_plan* P, int phase, const void* f_dev, void* u_dev, int nrhs, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (phase < 1 || phase > 6) return fail(LFDS_EINVAL, "phase must be 1..6");
  if (nrhs < 1 || !f_dev || !u_dev || !ws) return fail(LFDS_EINVAL, "bad solve arguments");
  if (P->opt.refine != 0) return fail(LFDS_EINVAL, "phased (sharded) solves do not refine");
  const int R = chunk_of(P, nrhs);
  if (R != nrhs) return fail(LFDS_EINVAL, "phased solves take all right-hand sides in one pass (rhs_chunk)");
  const int dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
  PassPlan* pp;
  int rc;
  if ((rc = get_pass(P, R, dt, dt, &pp))) return rc;
  if (ws_bytes < pp->total) return fail(LFDS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, pp->total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* w = reinterpret_cast<char*>(ws);
  Bufs b{};
  b.p[B_TAB] = P->d_tab;
  b.p[B_F] = const_cast<void*>(f_dev);
  b.p[B_U] = u_dev;
  b.p[B_MS] = w + pp->off_ms;
  b.p[B_T1] = w + pp->off_t1;
  b.p[B_IF] = w + pp->off_if;
  b.p[B_RED] = w + pp->off_red;
  b.p[B_CK] = w + pp->off_ck;
  (void)cudaGetLastError();  // (stale non-sticky errors of the caller)
  if (phase == 1) {
    P->launches = 0;
    CUDA_TRY(launch_fill_minpiv(reinterpret_cast<double*>(b.p[B_RED]), st));
  }
  const int ph = phase == 1 ? PH_1 : phase == 2 ? PH_2 : phase == 3 ? PH_3 : phase == 4 ? PH_2A : phase == 5 ? PH_2B
                                                                                                   : PH_INV;
  if ((rc = run_pass(P, *pp, b, R, dt, dt, st, ph))) return rc;
  P->report.passes = 1;
  P->report.n_kernel_launches = P->launches;
  if (phase == 3) {
    CUDA_TRY(cudaMemcpyAsync(P->h_piv, b.p[B_RED], sizeof(double), cudaMemcpyDeviceToHost, st));
    P->piv_stream = st;
    P->piv_pending = true;
  }
  return LFDS_OK;
}

static int solve_sharded_nccl(lfds_plan* P, const void* f_dev, void* u_dev, int nrhs, void* ws, size_t ws_bytes,
                              cudaStream_t st);

int lfds_solve(lfds_plan* P, const void* f_dev, void* u_dev, int nrhs, void* ws, size_t ws_bytes, void* stream) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (P->sharded && P->comm)  // block-sharded solve with the exchanges inside the library
    return solve_sharded_nccl(P, f_dev, u_dev, nrhs, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
  if (P->sharded) return fail(LFDS_EINVAL, "partitioned plan: use lfds_solve_phase with the two exchanges, or "
                                           "lfds_set_comm for in-library exchanges");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (nrhs < 1 || !f_dev || !u_dev || !ws) return fail(LFDS_EINVAL, "bad solve arguments");
  if (((uintptr_t)f_dev | (uintptr_t)u_dev | (uintptr_t)ws) & 15) return fail(LFDS_EINVAL, "pointers must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!P->opt.graph || P->opt.refine < 0) return solve_impl(P, f_dev, u_dev, nrhs, ws, ws_bytes, st);
  // CUDA graph: captured once per (f, u, nrhs, workspace) and replayed; the stage events of a
  // profiled plan are graph nodes, re-recorded by every replay
  const bool hit = P->gexec && P->gkey_f == f_dev && P->gkey_u == u_dev && P->gkey_ws == ws &&
                   P->gkey_wsb == ws_bytes && P->gkey_nrhs == nrhs;
  if (!hit) {
    // pending stage records of earlier replays refer to the old graph's events: drop_graph
    // takes their times before those events are destroyed
    drop_graph(P);
    // pass plans allocate device descriptors on first use: build them before capturing
    const int R = chunk_of(P, nrhs), dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
    for (int r0 = 0; r0 < nrhs; r0 += R) {
      PassPlan* pp;
      int rc;
      if ((rc = get_pass(P, std::min(R, nrhs - r0), dt, dt, &pp))) return rc;
      if (P->opt.refine != 0 && (rc = get_pass(P, std::min(R, nrhs - r0), 0, 0, &pp))) return rc;
    }
    // events already pending in the profile belong to earlier solves: keep them out of the graph
    const size_t nrec0 = P->prof.recs.size();
    if (!P->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeRelaxed));
    const int rc = solve_impl(P, f_dev, u_dev, nrhs, ws, ws_bytes, P->cap_stream);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(P->cap_stream, &g);
    if (rc) { if (g) cudaGraphDestroy(g); return rc; }
    CUDA_TRY(ce);
    const cudaError_t ie = cudaGraphInstantiate(&P->gexec, g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(ie);
    P->grecs.assign(P->prof.recs.begin() + nrec0, P->prof.recs.end());
    P->prof.recs.resize(nrec0);
    for (auto& r : P->grecs) r.graph = true;
    P->gkey_f = f_dev; P->gkey_u = u_dev; P->gkey_ws = ws; P->gkey_wsb = ws_bytes; P->gkey_nrhs = nrhs;
    P->grep = P->report;
  }
  CUDA_TRY(cudaGraphLaunch(P->gexec, st));
  P->report = P->grep;
  P->piv_stream = st;  // the graph ends with the monitor's copy into P->h_piv
  P->piv_pending = true;
  for (const auto& r : P->grecs) P->prof.recs.push_back(r);  // this replay's stage events
  return LFDS_OK;
}

static int solve_host_impl(lfds_plan* P, const void* f_host, void* u_host, int nrhs, void* ws, size_t ws_bytes,
                           void* stream, bool sync);

int lfds_solve_host(lfds_plan* P, const void* f_host, void* u_host, int nrhs, void* ws, size_t ws_bytes, void* stream) {
  return solve_host_impl(P, f_host, u_host, nrhs, ws, ws_bytes, stream, true);
}

int lfds_solve_host_async(lfds_plan* P, const void* f_host, void* u_host, int nrhs, void* ws, size_t ws_bytes,
                          void* stream) {
  return solve_host_impl(P, f_host, u_host, nrhs, ws, ws_bytes, stream, false);
}

static int solve_host_impl(lfds_plan* P, const void* f_host, void* u_host, int nrhs, void* ws, size_t ws_bytes,
                           void* stream, bool sync) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (nrhs < 1 || !f_host || !u_host || !ws) return fail(LFDS_EINVAL, "bad solve arguments");
  size_t need = lfds_workspace_bytes_host(P, nrhs);
  if (ws_bytes < need) return fail(LFDS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
  size_t el = P->opt.dtype == LFDS_F64 ? 8 : 16;
  size_t vol = (size_t)P->ax[0].N * P->ax[1].N * P->nz * nrhs * el;
  size_t base = lfds_workspace_bytes(P, nrhs);
  char* w = reinterpret_cast<char*>(ws);
  void* fd = w + base;
  void* ud = w + base + al256(vol);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaMemcpyAsync(fd, f_host, vol, cudaMemcpyHostToDevice, st));
  int rc = solve_impl(P, fd, ud, nrhs, ws, base, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(u_host, ud, vol, cudaMemcpyDeviceToHost, st));
  if (sync) CUDA_TRY(cudaStreamSynchronize(st));
  return LFDS_OK;
}

int lfds_residual(lfds_plan* P, const void* u_dev, const void* f_dev, lfds_z* r_dev, int nrhs, int dd, double* norms,
                  void* stream) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (!u_dev || nrhs < 1) return fail(LFDS_EINVAL, "bad residual arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
  double* d_norms = nullptr;
  if (norms) CUDA_TRY(cudaMallocAsync(&d_norms, sizeof(double) * 2 * nrhs, st));
  if (d_norms) CUDA_TRY(cudaMemsetAsync(d_norms, 0, sizeof(double) * 2 * nrhs, st));
  Bufs b{};
  b.p[B_TAB] = P->d_tab;
  const Axis& X = P->ax[0];
  const Axis& Y = P->ax[1];
  CUDA_TRY(launch_residual(X.N, Y.N, P->nz, nrhs, dt, dd, f_dev != nullptr, X.hoff, Y.hoff, P->t_hz, X.hhoff, Y.hhoff,
                           P->t_hhz, P->t_sig, P->t_sige, make_double2(P->lam.real(), P->lam.imag()), P->t_dd, u_dev,
                           f_dev,
                           reinterpret_cast<double2*>(r_dev), 0, d_norms, b, st));
  if (norms) {
    CUDA_TRY(cudaMemcpyAsync(norms, d_norms, sizeof(double) * 2 * nrhs, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int r = 0; r < nrhs; ++r) { norms[2 * r] = std::sqrt(norms[2 * r]); norms[2 * r + 1] = std::sqrt(norms[2 * r + 1]); }
    CUDA_TRY(cudaFree(d_norms));
  }
  return LFDS_OK;
}

int lfds_residual_f(lfds_plan* P, const void* u_dev, const void* f_dev, lfds_z* r_dev, int nrhs, int dd,
                    void* stream) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (!u_dev || !f_dev || !r_dev || nrhs < 1) return fail(LFDS_EINVAL, "bad residual arguments");
  (void)cudaGetLastError();  // (stale non-sticky errors of the caller)
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
  Bufs b{};
  b.p[B_TAB] = P->d_tab;
  const Axis& X = P->ax[0];
  const Axis& Y = P->ax[1];
  CUDA_TRY(launch_residual(X.N, Y.N, P->nz, nrhs, dt, dd, 1, X.hoff, Y.hoff, P->t_hz, X.hhoff, Y.hhoff, P->t_hhz,
                           P->t_sig, P->t_sige, make_double2(P->lam.real(), P->lam.imag()), P->t_dd, u_dev, f_dev,
                           reinterpret_cast<double2*>(r_dev), 1, nullptr, b, st));
  return LFDS_OK;
}

int lfds_axpy(lfds_plan* P, const lfds_z* delta_dev, void* u_dev, int nrhs, void* stream) {
  if (!P) return fail(LFDS_EINVAL, "plan is NULL");
  if (!P->d_tab) return fail(LFDS_ENODEVICE, "host-only plan (options.device < 0)");
  if (!delta_dev || !u_dev || nrhs < 1) return fail(LFDS_EINVAL, "bad axpy arguments");
  (void)cudaGetLastError();  // (stale non-sticky errors of the caller)
  const int dt = P->opt.dtype == LFDS_F64 ? 1 : 0;
  const int64_t n = (int64_t)P->ax[0].N * P->ax[1].N * P->nz * nrhs;
  CUDA_TRY(launch_axpy_u(n, dt, reinterpret_cast<const double2*>(delta_dev), u_dev,
                         reinterpret_cast<cudaStream_t>(stream)));
  return LFDS_OK;
}

int lfds_get_report(const lfds_plan* cP, lfds_report* rep) {
  if (!cP || !rep) return fail(LFDS_EINVAL, "NULL argument");
  lfds_plan* P = const_cast<lfds_plan*>(cP);
  if (P->piv_pending) {
    CUDA_TRY(cudaStreamSynchronize(P->piv_stream));
    P->report.min_pivot_ratio = *P->h_piv;
    if (P->gexec) P->grep.min_pivot_ratio = *P->h_piv;
    P->piv_pending = false;
  }
  *rep = P->report;
  if (rep->min_pivot_ratio >= 0 && rep->min_pivot_ratio < 1e-14)
    return fail(LFDS_ERESONANCE, "z-sweep pivot ratio %.3g < 1e-14 in the last solve (near-singular T_lm)",
                rep->min_pivot_ratio);
  return LFDS_OK;
}

int lfds_get_info(const lfds_plan* P, lfds_info* info) {
  if (!P || !info) return fail(LFDS_EINVAL, "NULL argument");
  *info = P->info;
  return LFDS_OK;
}

int lfds_get_basis(const lfds_plan* P, int axis, int block, int* n, int* kind, int* lo, lfds_z* lam, lfds_z* W) {
  if (!P || axis < 0 || axis > 1) return fail(LFDS_EINVAL, "bad axis");
  const Axis& A = P->ax[axis];
  const Basis* B;
  int l0 = 1;
  if (block < 0) {
    if (A.iface.empty()) {
      if (A.blocks.size() != 1) return fail(LFDS_EINVAL, "no global basis");
      B = &A.blocks[0].B;  // single block == global
    } else {
      B = &A.G;
    }
  } else {
    if (block >= (int)A.blocks.size()) return fail(LFDS_EINVAL, "block index out of range");
    B = &A.blocks[block].B;
    l0 = A.blocks[block].lo;
  }
  if (n) *n = B->n;
  if (kind) *kind = B->kind;
  if (lo) *lo = l0;
  if (lam) for (int i = 0; i < B->n; ++i) lam[i] = lfds_z{B->lam[i].real(), B->lam[i].imag()};
  if (W) for (size_t q = 0; q < (size_t)B->n * B->n; ++q) W[q] = lfds_z{B->W[q].real(), B->W[q].imag()};
  return LFDS_OK;
}

void lfds_destroy(lfds_plan* P) {
  if (!P) return;
  if (nccl().ok)
    for (NcclComm c : {P->comm_m, P->comm_l, P->comm})
      if (c) nccl().comm_destroy(c);
  for (auto& kv : P->passes) {
    free_pass(kv.second);
  }
  if (P->d_tab) cudaFree(P->d_tab);
  if (P->h_piv) cudaFreeHost(P->h_piv);
  if (P->gexec) cudaGraphExecDestroy(P->gexec);
  if (P->cap_stream) cudaStreamDestroy(P->cap_stream);
  for (auto& r : P->grecs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto& r : P->prof.recs)
    if (r.graph) continue;
    else { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : P->prof.pool) cudaEventDestroy(e);
  delete P;
}

}  // extern "C"
