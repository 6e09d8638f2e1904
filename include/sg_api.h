/*
 * sg_api.h -- C ABI of the sm_100a PCG / geometric-multigrid solver layer
 * (drop-in for the hot path of arXiv 2604.26441's reference package
 * `simpgmg`, /root/reference/pkg/src/simpgmg).
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch types.  Vector arguments are
 *     DEVICE pointers in the reference's free-DOF ordering (grid.py:3-8,
 *     free_dofs = flatnonzero(~mask)); FP64 vectors are double, FP32/BF16
 *     tagged vectors are float (fine_operator.py:68-77).
 *   - `stream` is a cudaStream_t passed as void*.
 *   - Every function returns 0 on success, nonzero on failure; the message is
 *     available from sg_last_error() (thread-local).  Solver failures are not
 *     errors: they are reported in sg_report.failure_kind (krylov.py:99-110).
 *   - Handles are internally serialized (one mutex each).
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef SG_API_H
#define SG_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sg_fine sg_fine; /* FineOperator (fine_operator.py:31-105) */
typedef struct sg_hier sg_hier; /* GmgHierarchy (hierarchy.py:181-216) */

enum { SG_TAG_FP64 = 0, SG_TAG_FP32 = 1, SG_TAG_BF16 = 2 }; /* precision.py:14-22 */
enum { SG_POLICY_FP64 = 0, SG_POLICY_FP32 = 1, SG_POLICY_BF16 = 2 }; /* hierarchy.py:52-56 */
enum { SG_FAIL_NONE = 0, SG_FAIL_CAP = 1, SG_FAIL_STAGNATION = 2, SG_FAIL_NON_FINITE = 3 };

const char* sg_last_error(void);
int sg_version(void);

/* ---------------------------------------------------------------------
 * Fine operator
 * ------------------------------------------------------------------- */
/* FineOperator.__init__ (fine_operator.py:34-47).  dof_mask: host bytes,
 * 3*(nx+1)*(ny+1)*(nz+1), nonzero = Dirichlet; NULL selects the cantilever
 * mask of build_cantilever (grid.py:141-162).  E: host, nx*ny*nz moduli.
 * ke: host row-major 24x24 unit element stiffness (element.py:23-70). */
int sg_fine_create(int nx, int ny, int nz, const uint8_t* dof_mask, const double* E,
                   const double* ke, sg_fine** out);
void sg_fine_destroy(sg_fine* op);
int64_t sg_fine_n_free(const sg_fine* op);
/* FineOperator.matvec_tagged (fine_operator.py:56-77); tag SG_TAG_*. */
int sg_fine_apply(sg_fine* op, int tag, const void* u_free, void* y_free, void* stream);
/* Same apply on NODE-layout device vectors (3*(nx+1)*(ny+1)*(nz+1), Dirichlet
 * entries zero): the raw kernel without the free<->node gather/scatter. */
int sg_fine_apply_nodes(sg_fine* op, int tag, const void* u_nodes, void* y_nodes, void* stream);
int64_t sg_fine_n_nodes(const sg_fine* op);
/* Number of kernel launches issued by the library so far (instrumentation). */
uint64_t sg_launch_count(void);
/* FineOperator.diagonal (fine_operator.py:79-86), floored. */
int sg_fine_diagonal(sg_fine* op, double* d_free, void* stream);
/* FineOperator.assemble_dense (fine_operator.py:88-101): device n_free^2. */
int sg_fine_dense(sg_fine* op, double* K, void* stream);
/* Distinct (child << 24 | fixed-local-dof mask) codes of fine elements that
 * touch Dirichlet DOFs (transfer.py:158-164), ascending; host output.
 * codes = NULL: size query (only *n is written). */
int sg_fine_boundary_codes(sg_fine* op, uint32_t* codes, int cap, int* n);

/* ---------------------------------------------------------------------
 * Hierarchy
 * ------------------------------------------------------------------- */
typedef struct {
  int levels;              /* requested depth (clamped at odd dims) */
  int policy;              /* SG_POLICY_* */
  int smoother_kind;       /* 0 chebyshev, 1 jacobi (smoothers.py:33-54) */
  int degree;
  double alpha;
  double omega;
  int coarse_smooth_steps;
  int cholesky_cutoff;
  int coarse_pcg_steps;
  uint64_t power_seed;
} sg_hier_params;

/* build_hierarchy (hierarchy.py:219-282).  triples: host 8x24x24 P_c^T Ke P_c
 * (transfer.py:143); codes/diffs: per boundary code, masked - triple
 * (transfer.py:161-164); lam_cache: per-level lambda_max to reuse (NULL). */
int sg_hier_create(sg_fine* op, const sg_hier_params* p, const double* triples,
                   const uint32_t* codes, const double* diffs, int ncodes,
                   const double* lam_cache, int n_cache, void* stream, sg_hier** out);
void sg_hier_destroy(sg_hier* h);

typedef struct {
  int n_levels;
  int clamped;        /* depth clamped at an odd dimension (hierarchy.py:252-259) */
  int coarsest_dense; /* 1 dense_cholesky, 0 pcg80 (hierarchy.py:123-136) */
  double eps;         /* max(mean_diag * 1e-8, 1e-14) */
} sg_hier_info;
int sg_hier_get_info(sg_hier* h, sg_hier_info* info);

typedef struct {
  int nx, ny, nz;
  int tag;
  int64_t n_free;
  int64_t nnz;        /* CSR nnz of the assembled operator (0 for level 0) */
  double lam_max;     /* 1.1 * power estimate (hierarchy.py:40-47) */
} sg_level_info;
int sg_hier_level_info(sg_hier* h, int level, sg_level_info* info);
/* Canonical CSR of an assembled level (transfer.py:33-39); host arrays sized
 * n_free+1 / nnz / nnz. */
int sg_hier_level_csr(sg_hier* h, int level, int64_t* indptr, int64_t* indices, double* data);
/* host bytes 3*(nx+1)*(ny+1)*(nz+1): the level's injected Dirichlet mask */
int sg_hier_level_mask(sg_hier* h, int level, uint8_t* dof_mask);
int sg_hier_level_diag(sg_hier* h, int level, double* diag_free, void* stream);
/* GmgHierarchy.vcycle (gamma 1) / wcycle (gamma 2) (hierarchy.py:199-216) */
int sg_hier_cycle(sg_hier* h, int gamma, const double* r_free, double* z_free, void* stream);
/* _Level.matvec64 / matvec_tagged (hierarchy.py:98-111) */
int sg_hier_level_apply(sg_hier* h, int level, int tag, const void* x_free, void* y_free,
                        void* stream);
/* _Level.smooth (hierarchy.py:113-120); x0_free may be NULL (zero guess) */
int sg_hier_level_smooth(sg_hier* h, int level, const double* b_free, const double* x0_free,
                         double* out_free, void* stream);
/* TransferPair.prolong / restrict (transfer.py:50-54) between level and level+1 */
int sg_hier_prolong(sg_hier* h, int level, const double* xc_free, double* xf_free, void* stream);
int sg_hier_restrict(sg_hier* h, int level, const double* xf_free, double* xc_free, void* stream);
/* CoarsestSolve.solve (hierarchy.py:133-136) */
int sg_hier_coarsest_solve(sg_hier* h, const double* r_free, double* x_free, void* stream);
/* TransferPair.P in canonical CSR (transfer.py:85-107); host arrays, call with
 * indices == NULL to get nnz in *nnz first. */
int sg_hier_transfer_csr(sg_hier* h, int level, int64_t* indptr, int64_t* indices, double* data,
                         int64_t* nnz);

/* Device time (ms, CUDA events, L2 flushed before each rep) of one hot-path
 * component: 0 fine apply FP32, 1 fine apply FP64, 2 level-1 SpMV FP64,
 * 3 coarsest solve, 4 full V-cycle, 5 fine apply BF16.  Bench instrumentation. */
int sg_hier_profile(sg_hier* h, int what, int reps, double* ms_avg, void* stream);

/* ---------------------------------------------------------------------
 * Standalone transfers and level-1 assembly (transfer.py)
 * ------------------------------------------------------------------- */
typedef struct sg_transfer sg_transfer;
/* build_transfer (transfer.py:68-107): fine grid + injected coarse grid;
 * fails on an odd dimension.  mask as in sg_fine_create (NULL = cantilever). */
int sg_transfer_create(int nx, int ny, int nz, const uint8_t* dof_mask, sg_transfer** out);
void sg_transfer_destroy(sg_transfer* t);
/* coarse Dirichlet mask by injection (transfer.py:75-83); host bytes */
int sg_transfer_coarse_mask(sg_transfer* t, uint8_t* dof_mask);
/* transpose 0: y = P x (prolong, transfer.py:50-51); 1: y = P^T x (restrict, :53-54) */
int sg_transfer_apply(sg_transfer* t, int transpose, const double* x_free, double* y_free,
                      void* stream);
/* P in canonical CSR; indices == NULL returns nnz only */
int sg_transfer_csr(sg_transfer* t, int64_t* indptr, int64_t* indices, double* data,
                    int64_t* nnz);
/* assemble_level1 (transfer.py:129-174) as canonical CSR, bit-identical to the
 * reference; two-phase: indices == NULL returns nnz only. */
int sg_level1_csr(sg_fine* op, const double* triples, const uint32_t* codes, const double* diffs,
                  int ncodes, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz);

/* triple_product (transfer.py:177-181) on ARBITRARY CSR inputs (host arrays,
 * int64 indices, stored order honoured): canonical CSR of P^T (K P) with
 * scipy csr_matmat summation order, bit-identical.  nf = rows of P = size of K,
 * nc = columns of P.  Fetch with sg_csr_result_get (Cp: nc+1, Cj/Cx: nnz). */
int sg_ptap_csr(int64_t nf, int64_t nc, const int64_t* Pp, const int64_t* Pj, const double* Px,
                const int64_t* Kp, const int64_t* Kj, const double* Kx, void** result,
                int64_t* nnz, void* stream);
int sg_csr_result_get(void* result, int64_t* Cp, int64_t* Cj, double* Cx);
void sg_csr_result_free(void* result);
/* Development instrumentation: pcg80 phase timestamps (ns) of step 10, out[8*block + k]
 * for every block (out: 8 x 256 int64; unused blocks 0). */
int sg_hier_pcg80_trace(sg_hier* h, long long* out, void* stream);

/* ---------------------------------------------------------------------
 * Outer solvers (krylov.py)
 * ------------------------------------------------------------------- */
typedef struct {
  double tol;
  int maxiter;
  int restart;
} sg_solver_cfg;
typedef struct {
  int converged;
  int iterations;
  double final_true_residual;
  int failure_kind; /* SG_FAIL_* */
  double wall_time;
} sg_report;
/* pcg(op.matvec, h.vcycle | flat Jacobi, b, cfg) (krylov.py:113-165, :284-288).
 * ktag: precision of apply_K (FineOperator.precision); h NULL => 1/diag.
 * history: host, >= maxiter doubles (relative recurrence residuals). */
int sg_pcg(sg_fine* op, int ktag, sg_hier* h, int gamma, const double* b_free, double* x_free,
           const sg_solver_cfg* cfg, sg_report* rep, double* history, void* stream);
/* fgmres(op.matvec, h.vcycle, b, cfg) (krylov.py:168-281) */
int sg_fgmres(sg_fine* op, int ktag, sg_hier* h, int gamma, const double* b_free, double* x_free,
              const sg_solver_cfg* cfg, sg_report* rep, double* history, void* stream);
/* lanczos_kappa_eff(v -> M(K_fp64 v), n, m, seed) (diagnostics.py:38-79): returns the
 * projected matrix H (host m*m, row-major) and the steps used. */
int sg_lanczos(sg_fine* op, sg_hier* h, int gamma, int m, uint64_t seed, double* H, int* used,
               int* partial, void* stream);

/* ---------------------------------------------------------------------
 * Multi-GPU slab partition (BASELINE.json north_star: fine and first coarse
 * levels slab-partitioned over the GPUs of one node, halo exchange and PCG dot
 * allreduce over NCCL, deeper levels gathered).  The
 * reference is single-process, so these extend pcg(op.matvec, h.vcycle, b,
 * cfg) (krylov.py:113-165, bench/runner.py:66-88) with per-rank z-slab
 * windows: every rank passes the same global b and receives the same global x.
 * Data movement between ranks is delegated to the host's sg_comm callbacks
 * (torch.distributed over NCCL in paper_2604_26441_b200/slab.py); each is
 * stream-ordered on `stream` and returns 0 on success.
 * ------------------------------------------------------------------- */
typedef struct {
  void* ctx;
  /* fill the ghost node planes of a window vector of slab level `level` */
  int (*halo)(void* ctx, int level, void* vec, int elem_bytes, void* stream);
  /* in-place sum over ranks of n device doubles, in rank order */
  int (*allreduce)(void* ctx, double* vals, int n, void* stream);
  /* owned planes of every rank's window vector `win` -> full-grid vector `full` */
  int (*allgather)(void* ctx, int level, const double* win, double* full, void* stream);
} sg_comm;
typedef struct sg_dist sg_dist;
/* planes: n_dist x {w0, w1, o0, o1} global node planes of this rank's window
 * [w0, w1] and owned range [o0, o1) on slab levels 0..n_dist-1 (n_dist 1 or 2). */
int sg_dist_create(sg_hier* h, int n_dist, const int32_t* planes, const sg_comm* comm,
                   void* stream, sg_dist** out);
void sg_dist_destroy(sg_dist* d);
/* Same slab handle on the DEVICE transport (sg_peer.cu): halos, rank-ordered
 * sums and allgathers are kernels that store into the peer ranks' mailboxes
 * (CUDA IPC mappings) and signal with system-scope release/acquire flags; no
 * host callback, and the distributed cycle is captured in a CUDA graph.
 * planes_all: world x n_dist x {w0, w1, o0, o1} (every rank's windows).
 * Replaces the host-callback transport (slab.py TorchSlabComm) of sg_dist_create. */
int sg_dist_create_peer(sg_hier* h, int n_dist, const int32_t* planes_all, int rank, int world,
                        void* stream, sg_dist** out);
/* This rank's mailbox: 64-byte cudaIpcMemHandle_t (handle_out may be NULL) and
 * its device address (for ranks sharing one process; base_out may be NULL). */
int sg_dist_peer_handle(sg_dist* d, void* handle_out, uint64_t* base_out);
/* Map every other rank's mailbox: handles = world x 64 bytes (IPC, other
 * processes) or bases = world device addresses (same process); one is NULL. */
int sg_dist_peer_open(sg_dist* d, const void* handles, const uint64_t* bases);
/* Free the replicated full-grid copies of the slab levels held by the
 * hierarchy (its single-GPU cycle then reports an error). */
int sg_dist_release_full(sg_dist* d, void* stream);
/* method 0 = pcg (krylov.py:113-165), 1 = fgmres (krylov.py:168-281), with
 * apply_K = op.matvec under ktag and apply_M = V (gamma 1) / W (gamma 2) cycle. */
int sg_dist_solve(sg_dist* d, int method, int ktag, int gamma, const double* b_free,
                  double* x_free, const sg_solver_cfg* cfg, sg_report* rep, double* history,
                  void* stream);
/* what 0: y = K_ktag x (fine_operator.py:56-77); what 1: y = cycle(x) (hierarchy.py:207-216) */
int sg_dist_apply(sg_dist* d, int what, int ktag, int gamma, const double* x_free, double* y_free,
                  void* stream);

/* ---------------------------------------------------------------------
 * Deterministic device vector kernels for the generic (callable) Krylov and
 * smoother paths.  dtype: 0 = double, 1 = float.  All FMA-free.
 * ------------------------------------------------------------------- */
int sg_vec_dot(int dtype, int64_t n, const void* a, const void* b, double* out_host, void* stream);
/* y = y + alpha * x */
int sg_vec_axpy(int dtype, int64_t n, double alpha, const void* x, void* y, void* stream);
/* y = x + beta * y */
int sg_vec_xpby(int dtype, int64_t n, const void* x, double beta, void* y, void* stream);
/* c = a - b */
int sg_vec_sub(int dtype, int64_t n, const void* a, const void* b, void* c, void* stream);
/* c = a * b (elementwise) */
int sg_vec_mul(int dtype, int64_t n, const void* a, const void* b, void* c, void* stream);
/* c = a * s */
int sg_vec_scale(int dtype, int64_t n, const void* a, double s, void* c, void* stream);
/* c = a / s */
int sg_vec_div(int dtype, int64_t n, const void* a, double s, void* c, void* stream);
/* BF16 round-to-nearest-even on FP32 bits (precision.py:25-48) */
int sg_vec_bf16(int64_t n, const float* a, float* b, void* stream);

/* ---------------------------------------------------------------------
 * Fixtures on the device
 * make_state (states.py:58-111) drawn into HBM from the splitmix64 stream
 * (prng.py:20-52): rho = device, nx*ny*nz doubles; kind = index into
 * STATE_KINDS (0 uniform, 1 binary, 2 checkerboard, 3 layered,
 * 4 random_floor, 5 mixed_near_void).  Bit-identical to the host generator.
 * ------------------------------------------------------------------- */
int sg_make_state(int kind, int nx, int ny, int nz, double vf, double floor_, uint64_t seed,
                  double* rho, void* stream);

/* ---------------------------------------------------------------------
 * Host-only work plans (no device needed; used by the CPU tests).
 * sg_plan_brick: pcg80 brick split of the coarsest node grid -> {sx, sy, sz}
 *   ({0,0,0}: no split fits, the contiguous-range kernel runs).
 * sg_plan_p32: level-0 FP32 apply tiling -> {P pairs per tile row, T x tiles,
 *   SX x-tile stride in nodes, R element rows per y tile, y tiles, kchunk node
 *   planes per z chunk, z chunks}.
 * ------------------------------------------------------------------- */
int sg_plan_brick(int nx, int ny, int nz, int nsm, int32_t* out3);
/* slab.py halo_pieces restated natively (sg_peer.cu): windows = world x
 * {w0, w1, o0, o1} of one level -> out = {src, dst, p0, p1} pieces, -1
 * terminated (cap = max pieces). */
int sg_plan_halo(int world, const int32_t* windows, int32_t* out, int cap);
int sg_plan_p32(int nx, int ny, int nz, int nsm, int32_t* out7);
/* sg_plan_p32 for an explicit block size nt (256: two CTAs per SM, the fused
 * smoother / residual applies' default when R >= 5; 512: one CTA per SM). */
int sg_plan_p32_bs(int nx, int ny, int nz, int nsm, int nt, int32_t* out7);

#ifdef __cplusplus
}
#endif

#endif /* SG_API_H */
