// Internal declarations shared by the .cu translation units.
#pragma once
#include "sg_common.cuh"
#include "sg_reduce.cuh"

namespace sg {

enum Tag : int { TAG_FP64 = 0, TAG_FP32 = 1, TAG_BF16 = 2 };

template <class T>
struct KeParam {
  T k[576];  // row-major 24x24 element matrix (symmetric)
};
struct KeDiag {
  double d[24];
};
// Nonzeros of (W Ke W)/64 in the tensor Walsh basis (sg_fine_walsh.cu)
template <class T>
struct KwParam {
  T v[45];
};
bool walsh_params(const double* ke, KwParam<double>& p64, KwParam<float>& p32);

// ---------------------------------------------------------------- fine level
struct FineOp {
  Grid grid;
  DBuf<double> E64;
  DBuf<float> E32;
  double ke_host[576];
  KeParam<double> ke64;
  KeParam<float> ke32;
  KeParam<float> ke16;  // bf16-rounded Ke32 (fine_operator.py:45)
  KeDiag kdiag;
  KwParam<double> kw64;
  KwParam<float> kw32;
  bool walsh_ok = false;
  double emax = 0.0;
  DBuf<float> p32a, p32b;  // P32 staging for node-layout FP32 applies (API path)
};

// FP64 / FP32 dispatch to the Walsh streaming kernel when the element matrix
// has the 45-entry Walsh pattern, else the dense node-centric kernel.
void fine_apply_f64(const FineOp& op, const double* u, double* y, cudaStream_t s);
void fine_apply_walsh_f32(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_walsh_f64(const FineOp& op, const double* u, double* y, cudaStream_t s);
// P32 layout (sg_fine_pk.cu): component-planar rows for level-0 FP32 vectors
int p32_xs(const GridDesc& g);
int64_t p32_size(const GridDesc& g);
bool p32_supported(const FineOp& op);
struct PkPlan {
  int P = 0, T = 1, SX = 0, R = 0, tilesy = 0, kchunk = 0, nch = 0;
  int nt = 512;  // block size
};
PkPlan pk_plan(const GridDesc& g, int nsm, int nt);
int pk_threads(const GridDesc& g, int mode);  // mode: 0 plain, 1 Chebyshev, 2 residual
void fine_apply_p32(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_p32_cheb(const FineOp& op, const float* x, float* xout, const float* b,
                         const float* dinv, float* d, float A, float AC, bool first, cudaStream_t s,
                         double* xout64 = nullptr);
void cheb_first0_p32(const GridDesc& g, const double* b64, const float* dinv, float c0, float* b32,
                     float* d, float* x, cudaStream_t s);
void fine_apply_p32_res(const FineOp& op, const float* x, const double* r64, double* out64,
                        cudaStream_t s);
template <class Tin>
void to_p32(const GridDesc& g, const Tin* src, float* dst, cudaStream_t s);
template <class Tout>
void from_p32(const GridDesc& g, const float* src, Tout* dst, cudaStream_t s);
int kKwRowHost(int q);
// fused FP64 stencil apply + Chebyshev step / residual (sg_stencil.cu)
void stencil_cheb64(const Grid& g, const double* At, const double* x, double* xout, const double* b,
                    const double* dinv, double* d, double A, double AC, bool first, cudaStream_t s);
// Symmetric (upper-slot) FP64 stencil copy and its SpMV (sg_stencil.cu):
// mode 0 y = A x, 1 fused Chebyshev step (as stencil_cheb64), 2 r - A x.
void stencil_sym_tile(const Grid& g, const double* A, DBuf<double>& Ts, cudaStream_t s);
void stencil_sym64(const Grid& g, const double* Ts, int mode, const double* x, double* out,
                   const double* b, const double* dinv, double* d, double A, double AC, bool first,
                   cudaStream_t s);
void stencil_res64(const Grid& g, const double* At, const double* x, const double* r, double* out,
                   cudaStream_t s);
int kKwColHost(int q);
bool p64_supported(const FineOp& op);
bool fine_apply_bf16_tc2(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_p64(const FineOp& op, const double* u, double* y, cudaStream_t s);
void make_state_device(int kind, int nx, int ny, int nz, double vf, double floor_,
                       unsigned long long seed, double* rho, cudaStream_t s);
void fine_apply_dense_f32(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_dense_f64(const FineOp& op, const double* u, double* y, cudaStream_t s);
void fine_apply_f32(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_bf16(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_bf16_tc(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_apply_bf16_dense(const FineOp& op, const float* u, float* y, cudaStream_t s);
void fine_diag_raw(const FineOp& op, double* d, cudaStream_t s);

// ------------------------------------------------------ grids and vectors
void build_grid(Grid& g, int nx, int ny, int nz, const uint8_t* dof_mask_host /*nullable*/,
                cudaStream_t s);
void build_coarse_grid(const Grid& fine, Grid& coarse, cudaStream_t s);
void build_window_grid(const Grid& full, int k0, int k1, Grid& win, cudaStream_t s);

template <class T>
void gather_free(const Grid& g, const T* node_vec, T* free_vec, cudaStream_t s);
template <class T>
void scatter_free(const Grid& g, const T* free_vec, T* node_vec, cudaStream_t s);
void cvt_f64_to_f32(int64_t n, const double* a, float* b, cudaStream_t s);
void cvt_f32_to_f64(int64_t n, const float* a, double* b, cudaStream_t s);

// numpy pairwise (np.add.reduce) mean over the free-ordered entries of a node
// vector, written to *out (device).  Bit-identical to numpy's float64 mean.
void np_mean_free(const Grid& g, const double* node_vec, double* out_dev, cudaStream_t s);
// d = max(d, 1e-14 * mean) on free dofs (fine_operator.py:86, hierarchy.py:88)
void diag_floor(const Grid& g, double* d, const double* mean_dev, cudaStream_t s);

// ------------------------------------------------------------- transfers
// x_f += P x_c (add = true) or x_f = P x_c; node layout, fixed entries zero.
void prolong(const Grid& fine, const Grid& coarse, const double* xc, double* xf, bool add,
             cudaStream_t s, float* xp32 = nullptr, int XS = 0);
void restrict_(const Grid& fine, const Grid& coarse, const double* xf, double* xc,
               cudaStream_t s);
void transfer_export_csr(const Grid& fine, const Grid& coarse, int64_t* indptr, int64_t* indices,
                         double* data, int64_t* nnz, cudaStream_t s);

// -------------------------------------------------- 27-point block stencils
// SoA storage: A[(slot*9 + ra*3 + cb) * nnodes + node], slot = (dk+1)*9+(dj+1)*3+(di+1).
struct Stencil {
  DBuf<double> A64;
  DBuf<float> A32;
  DBuf<double> T64;  // tiled copies for the SpMV (stencil_tile)
  DBuf<double> T64s;  // symmetric tiled copy (stencil_sym_tile), single-GPU FP64 levels
  DBuf<float> T32;
  int64_t nnz = 0;  // nonzero entries on free rows (CSR nnz of the reference)
};

// y = A x with At the tiled copy of A (stencil_tile)
template <class T>
void stencil_apply(const Grid& g, const T* At, const T* x, T* y, cudaStream_t s);
template <class T>
void stencil_tile(const Grid& g, const T* A, DBuf<T>& At, cudaStream_t s);
void stencil_diag(const Grid& g, const double* A, double* d, cudaStream_t s);
void stencil_round_f32(const Grid& g, const double* A64, float* A32, bool bf16, cudaStream_t s);
void fine_to_stencil(const FineOp& op, double* A, cudaStream_t s);
int64_t stencil_count_nnz(const Grid& g, const double* A, cudaStream_t s);
void stencil_export_csr(const Grid& g, const double* A, int64_t* indptr, int64_t* indices,
                        double* data, cudaStream_t s);
void stencil_to_dense(const Grid& g, const double* A, double* dense, double eps,
                      cudaStream_t s);

// level-1 Galerkin aggregation (transfer.py:129-174), bit-exact.
struct L1Tables {
  double tri[8 * 576];         // P_c^T Ke P_c (host numpy)
  std::vector<uint32_t> codes; // boundary codes: child<<24 | fixed-local-dof mask24
  std::vector<double> diffs;   // per code: masked - tri[child]
};
void boundary_codes(const FineOp& op, std::vector<uint32_t>& codes, cudaStream_t s);
void galerkin_level1(const FineOp& op, const Grid& coarse, const L1Tables& t, double* A,
                     cudaStream_t s);
// K_{l+1} = P^T K_l P with scipy csr_matmat summation order (transfer.py:177-181).
void galerkin_next(const Grid& fine, const Grid& coarse, const double* Af, double* Ac,
                   cudaStream_t s);

// ------------------------------------------------------------ misc kernels
void fill_gaussian_unit(const Grid& g, uint64_t seed, double* v_node, RedWork& w,
                        double* scratch_dev, cudaStream_t s);

}  // namespace sg
