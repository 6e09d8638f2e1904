// Hierarchy, cycle and solver orchestration (host C++ driving device kernels).
#pragma once
#include <memory>
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

// Scratch vectors of one level (node layout).
struct LevelWork {
  DBuf<double> r, x, d64, y64, dd64;
  DBuf<float> b32, x32, y32, dd32;
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
  LevelWork w;
  int64_t nd() const { return 3 * g->d.nnodes(); }
};

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
  ~Hier();
};
// One V/W-cycle from lv[0]->w.r into lv[0]->w.x, replayed from a CUDA graph
// captured on first use (set SG_NO_GRAPH=1 to launch kernel by kernel).
void cycle_run(Hier& H, int gamma, cudaStream_t s);

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
struct NativeSys {
  FineOp* fine;
  FineWork* fw;
  int ktag;      // tag of apply_K (FineOperator.precision)
  Hier* hier;    // nullptr => Jacobi (1/diag)
  int gamma;     // 1 V-cycle, 2 W-cycle
};

void pcg_native(NativeSys& sys, const double* b_node, double* x_node, const SolverCfg& cfg,
                SolveOut& out, std::vector<double>& hist, cudaStream_t s);
void fgmres_native(NativeSys& sys, const double* b_node, double* x_node, const SolverCfg& cfg,
                   SolveOut& out, std::vector<double>& hist, cudaStream_t s);
// Lanczos on v -> M(K v); returns H (m x m, row-major) and the number of steps used.
void lanczos_native(NativeSys& sys, int m, uint64_t seed, std::vector<double>& H, int& used,
                    bool& partial, cudaStream_t s);

}  // namespace sg
