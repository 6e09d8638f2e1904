// Hierarchy, cycle and solver orchestration (host C++ driving device kernels).
#pragma once
#include <array>
#include <memory>
#include <vector>
#include "sg_coarse.cuh"

namespace sg {

struct HParams {
  int levels = 4;
  int policy = 1;         // 0 fp64, 1 fp32, 2 bf16 (hierarchy.py:52-56)
  int smoother_kind = 0;  // 0 chebyshev, 1 jacobi
  int degree = 2;
  double alpha = 1.0 / 30.0;
  double omega = 0.5;
  int coarse_smooth_steps = 2;
  int cholesky_cutoff = 5000;
  int coarse_pcg_steps = 80;
  uint64_t power_seed = 0;
};

// Host callbacks that move slab data between ranks (multi-GPU slab
// partition; implemented over torch.distributed / NCCL by the host layer).
// All are stream-ordered on the stream they are given.
// Level codes of the exchanges: 0, 1 = slab levels in the node layout (doubles
// or floats per node plane 3 (nx+1)(ny+1)); kP32Level = level 0 in the P32
// layout (3 * XS * (ny+1) floats per node plane, sg_fine_pk.cu).
constexpr int kP32Level = 2;
struct CommHooks {
  void* ctx = nullptr;
  // fill the ghost node planes of a window vector of distributed level `level`
  int (*halo)(void* ctx, int level, void* vec, int elem_bytes, void* stream) = nullptr;
  // in-place sum over ranks of n device doubles, summed in rank order (same bits everywhere)
  int (*allreduce)(void* ctx, double* vals, int n, void* stream) = nullptr;
  // owned planes of every rank's window vector -> the full-grid vector, on every rank
  int (*allgather)(void* ctx, int level, const double* win, double* full, void* stream) = nullptr;
  void exchange(int level, const void* v, int eb, cudaStream_t s) const {
    if (halo(ctx, level, const_cast<void*>(v), eb, s)) throw Error("slab halo exchange failed");
  }
  void sum(double* v, int n, cudaStream_t s) const {
    if (allreduce(ctx, v, n, s)) throw Error("slab allreduce failed");
  }
  void gather(int level, const double* win, double* full, cudaStream_t s) const {
    if (allgather(ctx, level, win, full, s)) throw Error("slab allgather failed");
  }
};

// Scratch vectors of one level (node layout).
struct LevelWork {
  DBuf<double> r, x, d64, y64, dd64;
  DBuf<float> b32, x32, y32, dd32;
  DBuf<float> x32b;        // P32 level: ping-pong partner of x32 for the fused smoother
  float* xcur = nullptr;   // P32 level: buffer holding the smoother's last FP32 iterate
};

struct Level {
  int idx = 0;
  int tag = TAG_FP64;
  bool is_fine = false;
  Grid own;
  const Grid* g = nullptr;
  Stencil st;
  int kind = 0, degree = 2;
  double alpha = 1.0 / 30.0, omega = 0.5;
  double lam = 0.0;
  DBuf<double> diag, dinv;
  DBuf<float> dinv32;
  DBuf<float> dinv32p;  // P32 copy of dinv32 (p32 levels)
  LevelWork w;
  bool p32 = false;  // level-0 FP32 vectors in the P32 layout (sg_fine_pk.cu)
  int64_t nd() const { return 3 * g->d.nnodes(); }
  int64_t n32() const { return p32_size(g->d); }
};

struct DistPart;
struct Hier {
  FineOp* fine = nullptr;
  std::vector<std::unique_ptr<Level>> lv;
  int policy = 1;
  bool clamped = false;
  double emax = 0.0;
  int coarsest_mode = 1;  // 0 dense_cholesky, 1 pcg80
  double eps = 0.0;
  Pcg80 pcg;
  DenseInverse dense;
  RedWork red;
  DBuf<double> scal;  // device scalars
  DBuf<double> io_a, io_b;  // free<->node staging for the API (fine level)
  // CUDA graphs of the whole cycle (lv[0]->w.r -> lv[0]->w.x), per gamma
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  size_t graph_nodes[3] = {0, 0, 0};
  const CommHooks* comm = nullptr;  // slab windows: halo before every level apply
  DistPart* dist = nullptr;         // slab windows: the part (coarse-tail transition)
  bool released = false;  // slab levels freed for a slab solve (dist_release_full)
  // V-cycle variant for the native PCG on a P32 level: the final f64 output z is
  // not written (z = f64 of the FP32 iterate, read from P32 by rz_pupd)
  bool skip_z64 = false;
  cudaGraphExec_t graph_noz = nullptr;
  size_t graph_noz_nodes = 0;
  const float* zcur32 = nullptr;  // the noz graph's final FP32 iterate (P32 layout)
  ~Hier();
};
// One V/W-cycle from lv[0]->w.r into lv[0]->w.x, replayed from a CUDA graph
// captured on first use (set SG_NO_GRAPH=1 to launch kernel by kernel).
void cycle_run(Hier& H, int gamma, cudaStream_t s);
// V-cycle without the f64 output (level 0 in the P32 layout): returns the P32
// buffer holding z in FP32 (z_f64 = f64 of it exactly)
const float* cycle_run_noz(Hier& H, cudaStream_t s);

// Device scratch of the native solvers, allocated on first use and reused by
// every later solve (no cudaMalloc/cudaFree -- and their implicit device
// synchronisation -- inside a solve).
struct SolverWork {
  RedWork red;
  DBuf<double> sc;
  DBuf<float> t32a, t32b;
  DBuf<double> v[8];
  DBuf<double> basis1, basis2;
  DBuf<double> small;
  double* vec(int i, int64_t nd) {
    if (v[i].n < size_t(nd)) v[i].alloc(size_t(nd));
    return v[i].p;
  }
  static double* grow(DBuf<double>& b, size_t n) {
    if (b.n < n) b.alloc(n);
    return b.p;
  }
};

// Workspace attached to a fine operator for API-level applies.
struct FineWork {
  SolverWork sw;
  DBuf<double> u64, y64;
  DBuf<float> u32, y32;
  DBuf<double> diag;  // floored, node layout
  DBuf<double> dinv;  // 1/diag (0 on fixed), flat Jacobi preconditioner
  bool diag_ready = false;
  const double* diag_inv_ptr() const { return dinv.p; }
  RedWork red;
  DBuf<double> scal;
};

void fine_floored_diag(FineOp& op, FineWork& w, cudaStream_t s);
void fine_apply_tag(const FineOp& op, int tag, const void* x, void* y, cudaStream_t s);

std::unique_ptr<Hier> hier_build(FineOp* fine, FineWork& fw, const HParams& p, const L1Tables& t,
                                 const double* lam_cache, int n_cache, cudaStream_t s);
void level_apply(Hier& H, Level& L, int tag, const void* x, void* y, cudaStream_t s);
// smoother on level l: b, x0 (nullable) f64 node vectors -> out f64 node vector
void level_smooth(Hier& H, int l, const double* b, const double* x0, double* out, cudaStream_t s);
void cycle(Hier& H, int l, int gamma, cudaStream_t s);  // lv[l]->w.r -> lv[l]->w.x
void coarsest_solve(Hier& H, const double* r, double* x, cudaStream_t s);

// --------------------------------------------------------------- solvers
struct SolverCfg {
  double tol = 1e-6;
  int maxiter = 200;
  int restart = 32;
};
struct SolveOut {
  int converged = 0;
  int iterations = 0;
  double final_true_residual = 0.0;
  int failure_kind = 0;  // 0 none, 1 cap, 2 stagnation, 3 non_finite
  double wall_time = 0.0;
};

// Preconditioner / operator bundle for the native Krylov drivers.
struct DistPart;
struct NativeSys {
  FineOp* fine;
  FineWork* fw;
  int ktag;      // tag of apply_K (FineOperator.precision)
  Hier* hier;    // nullptr => Jacobi (1/diag)
  int gamma;     // 1 V-cycle, 2 W-cycle
  DistPart* dist = nullptr;  // slab-partitioned solve (fine = this rank's window)
};

// ------------------------------------------------------ multi-GPU slabs
// Device-side transport (sg_peer.cu): halo / rank-ordered sum / allgather as
// kernels storing into the peer ranks' IPC-mapped mailboxes.
struct PeerComm;
std::vector<std::array<int, 4>> halo_pieces(const std::vector<std::array<int, 4>>& win);
PeerComm* peer_create(int rank, int world, int n_dist, const int* planes_all, const int64_t* pnd,
                      const int* full_planes, int64_t p32_plane, cudaStream_t s, CommHooks& hooks);
void peer_destroy(PeerComm* p);
void peer_handle(PeerComm* p, void* out);
unsigned long long peer_base(PeerComm* p);
void peer_open(PeerComm* p, const void* handles, const unsigned long long* ptrs);

// One rank's part of a slab-partitioned hierarchy: levels 0..n_dist-1 are
// z-slab windows (owned node planes + ghost planes), the coarser levels are
// the replicated full hierarchy `full` (visited after an allgather of the
// cut level's residual).  Plane numbers are global node planes per level.
struct DistPart {
  int n_dist = 0;
  int w0[2] = {0, 0}, w1[2] = {0, 0}, o0[2] = {0, 0}, o1[2] = {0, 0};
  CommHooks comm;
  Hier* full = nullptr;
  FineOp wfine;                  // level-0 window operator
  FineWork wfw;                  // its solver scratch
  std::unique_ptr<Hier> W;       // window levels (W->lv[0] fine window, W->lv[1] L1 window)
  DBuf<double> bfull, xfull;     // full level-0 node vectors (API boundary)
  PeerComm* peer = nullptr;      // device transport (comm hooks point into it), or host hooks
  bool full_released = false;    // replicated slab levels of `full` freed (dist_release_full)
  // CUDA graphs of the distributed cycle (device transport only), per gamma
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  size_t graph_nodes[3] = {0, 0, 0};
  ~DistPart();
  int64_t plane_nd(int l) const { return 3 * int64_t(W->lv[size_t(l)]->g->d.nx + 1) * (W->lv[size_t(l)]->g->d.ny + 1); }
  int64_t own_off(int l) const { return (o0[l] - w0[l]) * plane_nd(l); }
  int64_t own_n(int l) const { return (o1[l] - o0[l]) * plane_nd(l); }
};
std::unique_ptr<DistPart> dist_build(Hier& full, int n_dist, const int* planes, const CommHooks& c,
                                     cudaStream_t s);
// one distributed V/W-cycle: W->lv[0]->w.r -> W->lv[0]->w.x
void dist_cycle(DistPart& D, int gamma, cudaStream_t s);
// the same, replayed from a CUDA graph when the transport is device-side
void dist_cycle_run(DistPart& D, int gamma, cudaStream_t s);
// free the replicated full-grid copies of the slab levels (stencils, work
// vectors) that the windows replaced; the coarse tail keeps what it reads
void dist_release_full(DistPart& D, cudaStream_t s);

void pcg_native(NativeSys& sys, const double* b_node, double* x_node, const SolverCfg& cfg,
                SolveOut& out, std::vector<double>& hist, cudaStream_t s);
void fgmres_native(NativeSys& sys, const double* b_node, double* x_node, const SolverCfg& cfg,
                   SolveOut& out, std::vector<double>& hist, cudaStream_t s);
void dist_apply(NativeSys& sys, int what, const double* xw, double* yw, cudaStream_t s);
// Lanczos on v -> M(K v); returns H (m x m, row-major) and the number of steps used.
void lanczos_native(NativeSys& sys, int m, uint64_t seed, std::vector<double>& H, int& used,
                    bool& partial, cudaStream_t s);

}  // namespace sg
