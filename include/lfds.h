/*
 * lfds.h — C ABI of the B200-native blocked separable Helmholtz solver
 * (layered-medium fast direct solver, arXiv 1909.01299, Druskin & Zaslavsky).
 *
 * Operation (Eq. (fd); Kronecker form Eq. (fdmtr) PAPER.md:38-40 with
 * reading R1 of DESIGN.md):  for unknown nodes (i,j,k), 1<=i<=nx, 1<=j<=ny, 1<=k<=nz,
 *
 *   sigma_k [ (u_{i+1}-u_i)/hx_i - (u_i-u_{i-1})/hx_{i-1} ] hy^_j hz^_k
 * + sigma_k [ (u_{j+1}-u_j)/hy_j - (u_j-u_{j-1})/hy_{j-1} ] hx^_i hz^_k
 * + [ sigma_{k+1/2}(u_{k+1}-u_k)/hz_k - sigma_{k-1/2}(u_k-u_{k-1})/hz_{k-1} ] hx^_i hy^_j
 * + lambda u hx^_i hy^_j hz^_k  =  f hx^_i hy^_j hz^_k,
 *
 * hd^_i = (hd_{i-1} + hd_i)/2, homogeneous Dirichlet on all six faces
 * (node 0 and node N+1 of every axis, reading R10).  lfds_solve returns the unique
 * solution u by the paper's two-level blocked separable method (steps 1-7)
 * on the device.  The method is direct: u = A^{-1} M f up to rounding.
 *
 * Data layout: fields f, u are [nrhs][nz][ny][nx] (x fastest), complex128 (interleaved
 * re,im == torch.complex128 == cuDoubleComplex), or float64 when the plan was created
 * with LFDS_F64 (all inputs real).
 *
 * Errors: every int-returning call returns an lfds_status; the message of the last error
 * on the calling thread is lfds_last_error().  Nothing is ever silently regularised
 * (SPEC S:303): a near-zero pivot is reported, not perturbed.
 */
#ifndef LFDS_H
#define LFDS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lfds_plan lfds_plan;            /* opaque; owned by the library */
typedef struct { double re, im; } lfds_z;      /* layout of complex128 */

typedef enum {
  LFDS_OK = 0,
  LFDS_EINVAL = 1,        /* bad sizes/steps/partition/pointers (see lfds_setup_grid) */
  LFDS_EEIG = 2,          /* 1D eigenbasis failed its residual / biorthonormality check */
  LFDS_ERESONANCE = 3,    /* z-system pivot below 1e-14 x row norm (lambda resonant) */
  LFDS_ENOMEM = 4,
  LFDS_ECUDA = 5,
  LFDS_ENCCL = 6,
  LFDS_ENOTCONVERGED = 7, /* refinement did not reach the requested residual */
  LFDS_ENODEVICE = 8      /* compute call on a host-only plan (options.device < 0) */
} lfds_status;

enum { LFDS_C128 = 0, LFDS_F64 = 1 };

typedef struct {
  int dtype;        /* LFDS_C128 or LFDS_F64 (real steps, sigma, lambda and f required)   */
  int refine;       /* refinement passes after the first solve pass: 0..8, or -1 = auto   */
                    /* (repeat while the residual improves 2x and exceeds refine_tol)     */
  double refine_tol;/* auto mode: stop when ||Au - Mf||/||Mf|| <= refine_tol (e.g. 1e-13)  */
  int residual_dd;  /* 1: refinement residual in double-double (reading R13), 0: fp64      */
  int device;       /* CUDA device ordinal; <0 = host-only plan (setup/basis queries only) */
  int rhs_chunk;    /* max right-hand sides processed per pipeline pass (0 = all)          */
  int profile;      /* 1: record CUDA events around every stage on the solve stream;       */
                    /* 2: also around every launch, per kernel kind (lfds_kernel_times)    */
  int s5_modal;     /* 1: step 5 with the z direction diagonalised too, when the z tables  */
                    /* are real (interface-only computation, no z sweeps);  */
                    /* 0: per-mode tridiagonal z-sweeps (the paper's form)   */
  int graph;        /* 1: lfds_solve captures its launches into a CUDA graph and replays  */
                    /* it while (f, u, nrhs, workspace) repeat (refine >= 0 only); 0: off */
  int plane_dst;    /* 1: steps 1 and 7 of a block that is uniform on both axes with the    */
                    /* same length n, 2(n+1) <= 128, run as ONE plane sine   */
                    /* transform (both axes, one pass over the block; longer blocks keep   */
                    /* the two passes); 0: always an x pass and a y pass;   */
                    /* lfds_info.n_plane_dst counts the blocks it applies to               */
  double resonance_tol; /* setup fails with LFDS_ERESONANCE when a block or the global family  */
                    /* of z-systems T_lm = A' + (lambda_l + mu_m) E has a relative margin   */
                    /* min|lambda_l + mu_m + theta_t| / (max|lambda_l| + max|mu_m| +        */
                    /* max|theta_t|) below this (reading R13; default 1e-13; <= 0: report   */
                    /* the margins in lfds_info without failing)                           */
  int zs_warp;      /* 1: step 2 with a warp per z-line (Thomas on 32 row chunks + parallel  */
                    /* cyclic reduction of the chunk separators across the lanes, tiles    */
                    /* staged in shared memory: one read and one write of v~    */
                    /* §6b); 0 (default): a thread per line (k_zs1, measured faster)        */
  int dst_tma;      /* 1 (default): the strided (y) sine passes load their tiles with TMA   */
                    /* tensor copies (k_dstt, one tensor map per block); 0: cp.async tiles */
} lfds_options;

/* Defaults: C128, refine 0, refine_tol 1e-13, residual_dd 1, device 0, rhs_chunk 0, s5_modal 1,
 * graph 0, plane_dst 1, resonance_tol 1e-13, zs_warp 0, dst_tma 1. */
void lfds_default_options(lfds_options* opt);

/*
 * Setup (timed separately from the solve; north_star): control volumes,
 * per-block and global 1D generalized eigenpairs A_d W = M_d W Lambda, W^T M_d W = I
 * (transpose reading R4), block classification (U = uniform real
 * steps -> exact sine modes; R = real; C = complex), z tables, device upload.
 *
 *  hx[nx+1], hy[ny+1], hz[nz+1]  host, complex steps h_0..h_N (h_t joins node t and t+1);
 *                                Re(h) > 0 required.
 *  sigma_node[nz]                host, sigma_k at nodes k = 1..nz (Re > 0).
 *  sigma_edge[nz+1]              host, sigma_{k+1/2} for k = 0..nz (Re > 0).
 *  lambda                        the shift of Eq. (wave2) (complex accepted, reading R11).
 *  if_x[n_if_x], if_y[n_if_y]    host, sorted 1-based interface nodes (width-1 planes,
 *                                reading R9); 2 <= node <= N-1, consecutive nodes >= 2 apart,
 *                                at most 32 per axis (33 blocks; more than 16 only with the
 *                                z-modal step 5, i.e. real z tables and options.s5_modal = 1).
 *                                n_if = 0 gives a single block (the global separable solve).
 *  opt                           may be NULL (defaults).
 *  *out                          receives the plan; release with lfds_destroy.
 * Returns LFDS_EINVAL on bad input, LFDS_EEIG if an eigenbasis fails its checks,
 * LFDS_ERESONANCE if a block's or the global z-systems are singular to within
 * opt->resonance_tol (the message names "global" or the block (i, j), the harmonic (l, m) and
 * the z-mode t; lfds_last_error), LFDS_ECUDA / LFDS_ENOMEM on device errors.  All host arrays
 * are only read.  (The margins are computed on the device: host-only plans report -1.)
 */
int lfds_setup_grid(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                    const lfds_z* sigma_node, const lfds_z* sigma_edge, lfds_z lambda,
                    int n_if_x, const int* if_x, int n_if_y, const int* if_y,
                    const lfds_options* opt, lfds_plan** out);

/* Device workspace (bytes, 256-B aligned) that lfds_solve needs for nrhs right-hand sides. */
size_t lfds_workspace_bytes(const lfds_plan* plan, int nrhs);

/*
 * Solve A u = M f for nrhs right-hand sides on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  f_dev, u_dev: device pointers, [nrhs][nz][ny][nx], 16-byte
 * aligned; u may alias f.  ws_dev: caller-owned device workspace of >= lfds_workspace_bytes.
 * Stream-ordered: the call returns after enqueueing, except in automatic refinement
 * (refine = -1), which reads residual norms back and so synchronises the stream.  The caller
 * owns f, u, ws.
 */
int lfds_solve(lfds_plan* plan, const void* f_dev, void* u_dev, int nrhs,
               void* ws_dev, size_t ws_bytes, void* cuda_stream);

/*
 * End-to-end variant with HOST buffers (pinned or pageable): copies f to the device
 * (inside ws: lfds_workspace_bytes_host), solves, copies u back, synchronises the stream.
 */
size_t lfds_workspace_bytes_host(const lfds_plan* plan, int nrhs);
int lfds_solve_host(lfds_plan* plan, const void* f_host, void* u_host, int nrhs,
                    void* ws_dev, size_t ws_bytes, void* cuda_stream);
/*
 * The same, enqueued only (returns before u_host is written; synchronise the stream).  With
 * pinned host buffers, separate workspaces and streams, consecutive solves overlap: the
 * host-to-device copy of one with the compute and device-to-host copy of the other.
 */
int lfds_solve_host_async(lfds_plan* plan, const void* f_host, void* u_host, int nrhs,
                          void* ws_dev, size_t ws_bytes, void* cuda_stream);

/*
 * Horizontally heterogeneous media — the paper's motivating use (large 3D
 * problems need iterative solvers, "the choice of preconditioner is crucial", preconditioning
 * "via discrete Green's function in layered medium").  Solves A_het u = M f where lambda varies
 * per node, lambda_ijk = lambda + dlam_ijk (Eq. (fd), with a node-wise lambda):
 *     A_het = A + diag(dlam) M.
 * Right-preconditioned restarted GMRES(restart) in the Lippmann-Schwinger (FDIE)
 * form  (I + diag(dlam) S) y = f,  u = S y,  with S = this plan's fast direct solve
 * (u = A^{-1} M f, lfds_solve), which equals M^{-1} A_het S exactly: one fast solve per
 * iteration, no stencil matvec.  Classical Gram-Schmidt with reorthogonalisation (CGS2).
 *   dlam_dev, f_dev, u_dev   device complex128 [nz][ny][nx], 16-B aligned; u_dev must not
 *                            alias f_dev or dlam_dev (nrhs = 1; complex128 plans only).
 *   tol                      stop when ||f - (I + dlam S) y||_2 <= tol ||f||_2 (> 0).
 *   maxit                    total iterations (>= 1); restart in 1..64.
 *   ws_dev                   >= lfds_gmres_workspace_bytes(plan, restart) (restart + 4 field
 *                            vectors, the solve workspace and reduction scratch).
 * Synchronises the stream (each Hessenberg column is read back).  The inner products are
 * per-CTA partial sums added on the host in a fixed order (deterministic).  Returns
 * LFDS_ENOTCONVERGED if maxit iterations do not reach tol (u then holds the last iterate).
 */
typedef struct {
  int iterations;          /* Arnoldi steps (= fast solves inside the iteration)            */
  int cycles;              /* restart cycles                                                 */
  double rel_residual;     /* ||f - (I + dlam S) y|| / ||f|| at exit (Arnoldi estimate)      */
} lfds_krylov_report;
size_t lfds_gmres_workspace_bytes(const lfds_plan* plan, int restart);
int lfds_gmres(lfds_plan* plan, const void* dlam_dev, const void* f_dev, void* u_dev, double tol, int maxit,
               int restart, void* ws_dev, size_t ws_bytes, void* cuda_stream, lfds_krylov_report* report);

/*
 * Residual r = M f - A u (b-units, PAPER.md Eq. (fdmtr)) on the device; f_dev may be NULL
 * (then r = -A u).  dd = 1 evaluates in double-double and rounds once.  r_dev is
 * complex128 [nrhs][nz][ny][nx] even for LFDS_F64 plans.  If norms != NULL it receives
 * 2*nrhs doubles (||r||_2, ||M f||_2 per rhs), which synchronises the stream.
 */
int lfds_residual(lfds_plan* plan, const void* u_dev, const void* f_dev, lfds_z* r_dev, int nrhs,
                  int dd, double* norms, void* cuda_stream);

/*
 * Refinement pieces for callers that run the passes themselves (block-sharded solves, whose
 * u is completed by a sum over the ranks between the passes; reading R13 of DESIGN.md):
 *  lfds_residual_f  r = f - M^{-1} A u in f-units (the right side whose solve is the correction
 *                   u_exact - u), device pointers, stream-ordered, no synchronisation; u_dev and
 *                   f_dev in the plan dtype, r_dev complex128 [nrhs][nz][ny][nx]; dd = 1
 *                   evaluates in double-double.
 *  lfds_axpy        u += delta over nrhs fields (u in the plan dtype: the real part is added for
 *                   LFDS_F64 plans), stream-ordered.
 * Errors: LFDS_EINVAL (NULL pointers, nrhs < 1), LFDS_ENODEVICE, LFDS_ECUDA.
 */
int lfds_residual_f(lfds_plan* plan, const void* u_dev, const void* f_dev, lfds_z* r_dev, int nrhs, int dd,
                    void* cuda_stream);
int lfds_axpy(lfds_plan* plan, const lfds_z* delta_dev, void* u_dev, int nrhs, void* cuda_stream);

/*
 * Block sharding across ranks (BASELINE.json north_star: "partitioned across the 8 B200s by
 * blocks S^ij, with NCCL over NVLink only for the interface exchange").  Every rank builds the
 * same plan, then lfds_set_partition tells it which blocks it computes in the two block passes
 * (steps 1-3, 6-7), which global x-modes l in [l_begin, l_end) it
 * sweeps in step 5, and whether it is the rank (exactly one) that adds the
 * b = M f terms of the step-4 residual and writes u on the interface planes.
 *  block_owned[nbx*nby]  host, row-major [block_y][block_x], nonzero = computed here;
 *                        NULL restores the unpartitioned plan.
 * A solve is then three phases on the caller's stream, with two sums over the ranks:
 *   lfds_solve_phase(1) -> sum exchange 1 over ranks (in place, e.g. NCCL all-reduce)
 *   lfds_solve_phase(2) -> sum exchange 2 over ranks
 *   lfds_solve_phase(3)
 * lfds_exchange_layout gives each exchange's byte offset inside the workspace and its length
 * in doubles (exchange 1 = the interface residual on the planes, exchange 2 = the step-5
 * correction projected onto the planes; exchange 3 = [R1~, R2~], see lfds_set_formation_rows).  Afterwards u_dev holds u on this rank's blocks and
 * on its segments of the interface planes (the segment of an x-plane in a block row belongs to
 * the owner of the block on its left, of a y-plane in a block column to the owner of the block
 * below, the plane intersections to the rank0 rank); other entries are not written.  Phased
 * solves take all nrhs right-hand sides in one pass and do not refine (LFDS_EINVAL otherwise):
 * a caller refines by summing u over the ranks, then lfds_residual_f, a phased solve of the
 * residual, a sum of the correction and lfds_axpy (paper_1909_01299_b200/dist.py).
 */
int lfds_set_partition(lfds_plan* plan, const int* block_owned, int l_begin, int l_end, int rank0);
/*
 * Optional second split of the z-modal step 5 (options.s5_modal, real z tables): this rank
 * forms the global y-modes m in [m_begin, m_end) (multiples of 64, the k_s5m tile, or ny) of
 * its x-modes, so R1 = W_y^T RX is formed only for those m; exchange 2 sums the (m, l) parts.
 * Call after lfds_set_partition (which resets it to all m).  LFDS_EINVAL for a bad or unaligned
 * range or when step 5 runs as per-mode z-sweeps.
 */
int lfds_set_mode_rows(lfds_plan* plan, int m_begin, int m_end);
/*
 * Formation split of the z-modal step 5 (after lfds_set_mode_rows): this rank FORMS only the
 * rows m in [m_begin, m_end) of R1~ = Z^T W_y^T RX and l in [l_begin, l_end) of R2~ (its share of
 * the plane transforms of the ranks that read the same rows), the other rows are zero, and a
 * third exchange sums [R1~, R2~] over the ranks (lfds_exchange_layout(3)).  The solve then runs
 * phase 1, exchange 1, phase 4 (step 5 up to R~), exchange 3, phase 5 (the modal solve and the
 * projections), exchange 2, phase 3; lfds_solve_phase(2) still runs 4 and 5 together.
 * m_begin < 0 switches it off.  LFDS_EINVAL without a partition or the z-modal step 5.
 */
int lfds_set_formation_rows(lfds_plan* plan, int m_begin, int m_end, int l_begin, int l_end);
int lfds_exchange_layout(const lfds_plan* plan, int nrhs, int which, size_t* byte_offset, size_t* n_doubles);
/*
 * In-library exchanges (BASELINE.json north_star: "NCCL over NVLink only for the interface
 * exchange"; PAPER.md:69-70 is that exchange).  NCCL is loaded at run time (dlopen of the
 * libnccl.so.2 already in the process, else the system one; LFDS_NCCL_LIB overrides): the
 * library links none.  One rank calls lfds_nccl_unique_id and the caller broadcasts the 128
 * bytes; then every rank of the group calls lfds_set_comm (collective, like ncclCommInitRank)
 * on its partitioned plan.  From then on lfds_solve on that plan runs the three phases with the
 * two exchanges summed by ncclAllReduce (float64, in place in the workspace) on the solve stream:
 * no host round trip between the phases.  id = NULL releases the communicator (back to
 * lfds_solve_phase + caller-driven sums).  LFDS_ENCCL if NCCL is missing or fails.
 */
int lfds_nccl_unique_id(unsigned char* id);  /* id: 128 bytes */
int lfds_set_comm(lfds_plan* plan, const unsigned char* id, int rank, int world);
/* Exchange-3 groups (collective over the communicator, ncclCommSplit): ranks with the same
 * color_m share their y-mode range (R1~ rows), the same color_l their x-mode range (R2~ rows);
 * exchange 3 then sums each half over its group only.  Without it, over all ranks. */
int lfds_set_comm_groups(lfds_plan* plan, int color_m, int color_l);
int lfds_solve_phase(lfds_plan* plan, int phase, const void* f_dev, void* u_dev, int nrhs, void* ws,
                     size_t ws_bytes, void* cuda_stream);

typedef struct {
  int passes;                  /* solve passes in the last lfds_solve (1 + refinements)     */
  double rel_residual[9];      /* refine = -1 (auto): ||Au-Mf||/||Mf|| before each refinement    */
                               /* pass and after the last (max over rhs); -1 = not read back     */
  double min_pivot_ratio;      /* min |pivot| / row-norm over all z-sweeps of the last call  */
                               /* (copied stream-ordered into pinned host memory at the end of */
                               /* the solve; lfds_get_report waits for that copy)              */
  int n_kernel_launches;       /* kernels enqueued by the last lfds_solve                   */
} lfds_report;
/* Synchronises the last solve's stream (for min_pivot_ratio).  Returns LFDS_ERESONANCE (and still
 * fills *rep) when min_pivot_ratio < 1e-14: an unpivoted z-sweep met a near-zero pivot and the
 * last solve must not be trusted (reported, never perturbed). */
int lfds_get_report(const lfds_plan* plan, lfds_report* rep);

typedef struct {
  int nx, ny, nz;
  int nbx, nby;                /* blocks per axis                                          */
  int n_if_x, n_if_y;
  int real_z;                  /* 1 if the z tables are real                                */
  double setup_seconds;        /* host wall time of lfds_setup_grid                          */
  double eig_max_residual;     /* max over all bases of ||AW-MWL||/(||A|| ||W||)              */
  double eig_max_biorth;       /* max over all bases of ||W^T M W - I||_max                   */
  size_t device_table_bytes;
  int s5_modal;                /* 1 if step 5 runs in the z-modal form (options.s5_modal, real z) */
  double z_eig_residual;       /* z modal basis: max|A'z - theta E z| / (||A'|| max|Z|)       */
  double z_eig_orth;           /* z modal basis: max|Z^T E Z - I|                             */
  int n_plane_dst;             /* blocks whose steps 1 and 7 run as one plane sine transform  */
                               /* (options.plane_dst; uniform on both axes, one length L <= 128,
                                  complex data)                                              */
  /* resonance margins (reading R13): min over (l, m, t) of |lambda_l + mu_m + theta_t|, theta_t
     the eigenvalues of the z pencil A' z = theta E z (ascending Re, then Im), lambda_l / mu_m in
     each basis' order (lfds_get_basis); 0-based indices; _rel divides by max|lambda_l| +
     max|mu_m| + max|theta_t| of the family; -1 if not computed (host-only plan)             */
  double margin_global, margin_global_rel;  /* step-5 global z-systems (single block: = block) */
  int margin_global_lmt[3];
  double margin_block, margin_block_rel;    /* the worst block's z-systems (steps 2 and 6)     */
  int margin_block_ij[2];                   /* that block (x index, y index)                   */
  int margin_block_lmt[3];
  int global_fold;             /* bit 0 / bit 1: the global x / y steps are palindromic, so the  */
                               /* step-5 plane transforms along that axis run on folded data at  */
                               /* half length (even / odd modes)                  */
  int n_plane_dense;           /* blocks whose steps 1 and 7 run as one plane  */
                               /* transform on DMMA (k_xplane): at most 32 nodes on both axes,    */
                               /* neither axis on the fast sine transform, complex data          */
                               /* and those blocks holding at least half of the block unknowns   */
                               /* (0 otherwise; the environment variable LFDS_XPLANE=0 forces the */
                               /* x pass + y pass form for A/B runs)              */
} lfds_info;
int lfds_get_info(const lfds_plan* plan, lfds_info* info);

/*
 * Basis query (for tests): axis 0 = x, 1 = y; block = -1 for the global basis, else the
 * block index along that axis.  *n receives the size; kind receives 0 = U (sine), 1 = R
 * (real), 2 = C (complex); lam (n) and W (n*n, row-major W[p*n + l]) may be NULL.
 */
int lfds_get_basis(const lfds_plan* plan, int axis, int block, int* n, int* kind, int* lo,
                   lfds_z* lam, lfds_z* W);

/*
 * Stage timing (options.profile = 1): device milliseconds per pipeline stage, measured with
 * CUDA events recorded on the solve stream around each stage, accumulated over all solves
 * since the previous call (which this call resets; it synchronises those events).
 * ms[i] and launches[i] for i < lfds_stage_count(); names from lfds_stage_name(i).
 */
int lfds_stage_count(void);
const char* lfds_stage_name(int stage);
int lfds_stage_times(lfds_plan* plan, double* ms, int* launches);

/*
 * Kernel timing (options.profile = 2): the same CUDA-event accounting per kernel KIND
 * (k_xform3m, k_zs1, ...; names from lfds_kernel_name), events recorded around every launch
 * of that kind on the solve stream; accumulated since the previous call, which resets them.
 */
int lfds_set_profile(lfds_plan* plan, int level);  /* 0, 1 or 2 (options.profile) for later solves */
int lfds_kernel_count(void);
const char* lfds_kernel_name(int kernel);
int lfds_kernel_times(lfds_plan* plan, double* ms, int* launches);

/*
 * In-run FP64 peak of the current device (roofline denominator of the DMMA-bound kernels):
 * a back-to-back mma.sync.m8n8k4.f64 (DMMA) loop on every SM, timed with CUDA events on
 * `cuda_stream` (synchronises it).  *tflops = 2 x FMA / s.  Returns LFDS_ECUDA on failure.
 */
int lfds_fp64_peak(void* cuda_stream, double* tflops);

void lfds_destroy(lfds_plan* plan);
const char* lfds_last_error(void);
const char* lfds_version(void);

/*
 * Multi-level (nested) partition — PAPER.md:77-79 (remark: "multiple mutually embedded
 * partitions of S" trade the global interface step for solves on each level of embedding).
 * Three levels: coarse blocks C between the coarse interfaces (c_x, c_y) and, inside every C,
 * fine blocks between the fine interfaces (f_x, f_y, a superset of c_x, c_y).  Every coarse-block
 * Dirichlet problem (PAPER.md:66-67 and :71-72 on the coarse partition) is solved by the
 * two-level method of its own fine partition, whose interface step uses C's eigenbases; only the
 * coarse planes take the global step 5.  A solve is
 *   v_C = A_C^{-1} M f_C;  r_b = M f - A v on the coarse planes;  w = step 5 (global bases);
 *   u_C = A_C^{-1} (M f_C - A_{C,dC} w);  u = w on the coarse planes,
 * exact up to rounding like the two-level method (u = A^{-1} M f).  Arguments as
 * lfds_setup_grid; c_x / c_y follow its interface rules, every one must be in f_x / f_y.
 * Complex128 device plans only, no refinement (LFDS_EINVAL otherwise).
 *  lfds_ml_solve: f_dev, u_dev device complex128 [nz][ny][nx] (one right-hand side), 16-byte
 *  aligned; ws_dev of at least lfds_ml_workspace_bytes; everything stream-ordered on
 *  cuda_stream.  The coarse-block plans replay as CUDA graphs (constant buffers).
 * Errors: the codes of lfds_setup_grid / lfds_solve, message in lfds_ml_last_error().
 */
typedef struct lfds_ml lfds_ml;
int lfds_ml_setup(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                  const lfds_z* sigma_node, const lfds_z* sigma_edge, lfds_z lambda,
                  int n_cx, const int* c_x, int n_cy, const int* c_y,
                  int n_fx, const int* f_x, int n_fy, const int* f_y,
                  const lfds_options* opt, lfds_ml** out);
size_t lfds_ml_workspace_bytes(const lfds_ml* ml);
int lfds_ml_solve(lfds_ml* ml, const void* f_dev, void* u_dev, void* ws_dev, size_t ws_bytes, void* cuda_stream);
int lfds_ml_get_plans(const lfds_ml* ml, int* n_coarse_blocks);
void lfds_ml_destroy(lfds_ml* ml);
const char* lfds_ml_last_error(void);

/*
 * Lebedev-grid Maxwell solve in a horizontally layered medium — PAPER.md §3 (lines 81-372).
 * Solves A_h H = f with A_h H = curl_h(rho curl_h H) - i omega mu H (Eq. (abstr), the curls
 * built from Eq. (fin)), rho = diag(c1, c2, c3)(z) (diagonal),
 * H on the Lebedev P-grid, boundary conditions H x n = 0 on dOmega ∩ P, E x n = 0 on dOmega ∩ R
 * (PAPER.md:238-241), by the paper's separable route: x/y transforms of the four families pp, dd
 * (even levels), pd, dp (odd levels) in the primary (Dirichlet) / dual (Neumann) eigenbases
 * (PAPER.md:248-268), per harmonic four decoupled systems with H_z eliminated, i.e. 2x2
 * block-tridiagonal z-systems, inverse transforms.  Exact up to rounding.
 *  nx, ny, nz   node counts N of the grid M (odd, >= 5; nodes 0..N-1, both ends on dOmega and
 *               primary, reading M1); hx[nx-1] ... steps x_{t+1} - x_t (complex
 *               steps = coordinate stretching, e.g. a PML).
 *  c1, c2, c3   rho = diag(c1, c2, c3) per z node (nz values each; used on the R nodes).
 *  mu, omega    permeability (complex allowed) and angular frequency (> 0).
 *  device       CUDA device; profile = 1 records CUDA events around the seven launch groups of
 *               every solve (lfds_mw_kernel_times; synchronises the stream after each solve).
 * Field layout (f, H, r): device complex128 [3][nz][ny][nx] (component x, y, z; x fastest),
 * 16-byte aligned; values are taken / written on the interior P nodes (i + j + k even, 0-based),
 * H and r are 0 elsewhere, f is ignored elsewhere.  Stream-ordered on cuda_stream.
 * Errors: LFDS_EINVAL (bad sizes / NULL / even N), LFDS_EEIG (an axis basis failed its checks),
 * LFDS_ERESONANCE (c2 lambda_l^2 + c1 nu_m^2 - i omega mu within 1e-13 of 0: the H_z
 * elimination is singular; the message names (l, m) and the level), LFDS_ECUDA / LFDS_ENOMEM.
 * Message in lfds_mw_last_error().
 */
typedef struct lfds_mw lfds_mw;
int lfds_mw_setup(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                  const lfds_z* c1, const lfds_z* c2, const lfds_z* c3, lfds_z mu, double omega,
                  int device, int profile, lfds_mw** out);
size_t lfds_mw_workspace_bytes(const lfds_mw* plan);
int lfds_mw_solve(lfds_mw* plan, const void* f_dev, void* h_dev, void* ws_dev, size_t ws_bytes, void* cuda_stream);
/* r = f - A_h H on the interior P nodes (0 elsewhere), evaluated directly on the grid (the same
 * workspace; its first 3 nz ny nx complex128 hold E = rho curl_h H afterwards). */
int lfds_mw_residual(lfds_mw* plan, const void* h_dev, const void* f_dev, void* r_dev, void* ws_dev,
                     size_t ws_bytes, void* cuda_stream);
int lfds_mw_kernel_count(void);
const char* lfds_mw_kernel_name(int kernel);
int lfds_mw_kernel_times(lfds_mw* plan, double* ms, int* launches);  /* accumulated; resets */
void lfds_mw_destroy(lfds_mw* plan);
const char* lfds_mw_last_error(void);

/*
 * Two-level (blocked) Maxwell solve, H = H^1 + H^2: blocks S^ij between the
 * x-interfaces ix[] and y-interfaces iy[] (node indices, even, >= 4 apart and >= 4 from the
 * ends, so every block is a Lebedev sub-grid with primary boundary nodes).  H^1 = block solves
 * with H x n = 0 on dS ∩ P, E x n = 0 on dS ∩ R (each block its own layered plan); the residual
 * f - A_h H^1 lives on the three node layers around each plane; step 5 evaluates A_h^{-1} of it on
 * those layers only (layer-restricted global transforms + all harmonics' 2x2 block z-systems);
 * the interface data H_tan (plane P nodes) and E_tan (plane R nodes) are lifted into the block
 * right sides and the blocks are solved again ("the boundary conditions are imposed on both
 * these grids").  Exact up to rounding.  Arguments and field layout as
 * lfds_mw_setup / lfds_mw_solve; errors in lfds_mw_last_error().
 */
typedef struct lfds_mw2 lfds_mw2;
int lfds_mw2_setup(int nx, const lfds_z* hx, int ny, const lfds_z* hy, int nz, const lfds_z* hz,
                   const lfds_z* c1, const lfds_z* c2, const lfds_z* c3, lfds_z mu, double omega,
                   int n_ix, const int* ix, int n_iy, const int* iy, int device, lfds_mw2** out);
size_t lfds_mw2_workspace_bytes(const lfds_mw2* plan);
int lfds_mw2_solve(lfds_mw2* plan, const void* f_dev, void* h_dev, void* ws_dev, size_t ws_bytes, void* cuda_stream);
int lfds_mw2_blocks(const lfds_mw2* plan, int* n_blocks);
void lfds_mw2_destroy(lfds_mw2* plan);

#ifdef __cplusplus
}
#endif
#endif /* LFDS_H */
