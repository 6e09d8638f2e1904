// Grids, free<->node conversions, numpy-exact pairwise mean, seeded start vectors.
#include <cmath>
#include "sg_kernels.cuh"

namespace sg {

// ------------------------------------------------------------------ grids
static void finish_grid(Grid& g, cudaStream_t s) {
  const GridDesc& d = g.d;
  const int64_t nn = d.nnodes();
  std::vector<int32_t> f2d, d2f(size_t(3 * nn), -1);
  f2d.reserve(size_t(3 * nn));
  bool xface = true;
  for (int64_t node = 0; node < nn; ++node) {
    const int i = int(node % (d.nx + 1));
    const uint8_t m = g.h_nmask[node];
    if ((i == 0 && m != 7) || (i != 0 && m != 0)) xface = false;
    for (int a = 0; a < 3; ++a) {
      if (!((m >> a) & 1)) {
        d2f[size_t(3 * node + a)] = int32_t(f2d.size());
        f2d.push_back(int32_t(3 * node + a));
      }
    }
  }
  SG_REQUIRE(3 * nn < (int64_t(1) << 31), "grid too large for int32 dof indices");
  g.d.xface = xface;
  g.n_free = int64_t(f2d.size());
  g.nmask.alloc(size_t(nn));
  g.nmask.upload(g.h_nmask.data(), size_t(nn), s);
  g.free2dof.alloc(f2d.size());
  g.free2dof.upload(f2d.data(), f2d.size(), s);
  g.dof2free.alloc(d2f.size());
  g.dof2free.upload(d2f.data(), d2f.size(), s);
  SG_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
}

void build_grid(Grid& g, int nx, int ny, int nz, const uint8_t* dof_mask, cudaStream_t s) {
  SG_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "element counts must be positive");
  g.d.nx = nx;
  g.d.ny = ny;
  g.d.nz = nz;
  const int64_t nn = g.d.nnodes();
  g.h_nmask.assign(size_t(nn), 0);
  for (int64_t node = 0; node < nn; ++node) {
    if (dof_mask) {
      uint8_t m = 0;
      for (int a = 0; a < 3; ++a) m |= uint8_t((dof_mask[3 * node + a] ? 1 : 0) << a);
      g.h_nmask[node] = m;
    } else {
      g.h_nmask[node] = (node % (nx + 1) == 0) ? 7 : 0;  // cantilever (grid.py:151-156)
    }
  }
  finish_grid(g, s);
}

// Slab window of a grid: node planes [k0, k1] (inclusive) of `full`, i.e. the
// element layers [k0, k1) with the same Dirichlet bits (multi-GPU slabs).
void build_window_grid(const Grid& full, int k0, int k1, Grid& w, cudaStream_t s) {
  SG_REQUIRE(0 <= k0 && k0 < k1 && k1 <= full.d.nz, "bad slab window");
  w.d.nx = full.d.nx;
  w.d.ny = full.d.ny;
  w.d.nz = k1 - k0;
  const int64_t plane = int64_t(full.d.nx + 1) * (full.d.ny + 1);
  w.h_nmask.assign(full.h_nmask.begin() + k0 * plane, full.h_nmask.begin() + (k1 + 1) * plane);
  finish_grid(w, s);
}

// Injection: coarse DOF fixed iff fine DOF at node (2i,2j,2k) is (transfer.py:75-83).
void build_coarse_grid(const Grid& fine, Grid& c, cudaStream_t s) {
  SG_REQUIRE(fine.d.nx % 2 == 0 && fine.d.ny % 2 == 0 && fine.d.nz % 2 == 0,
             "odd dimension cannot be coarsened");
  c.d.nx = fine.d.nx / 2;
  c.d.ny = fine.d.ny / 2;
  c.d.nz = fine.d.nz / 2;
  const int64_t nn = c.d.nnodes();
  c.h_nmask.assign(size_t(nn), 0);
  const int FX = fine.d.nx + 1, FY = fine.d.ny + 1;
  for (int k = 0; k <= c.d.nz; ++k)
    for (int j = 0; j <= c.d.ny; ++j)
      for (int i = 0; i <= c.d.nx; ++i) {
        const int64_t cn = i + int64_t(c.d.nx + 1) * (j + int64_t(c.d.ny + 1) * k);
        const int64_t fn = 2 * i + int64_t(FX) * (2 * j + int64_t(FY) * 2 * k);
        c.h_nmask[cn] = fine.h_nmask[fn];
      }
  finish_grid(c, s);
}

// ----------------------------------------------------------- conversions
template <class T>
__global__ void gather_kernel(int64_t n, const int32_t* __restrict__ f2d, const T* __restrict__ a,
                              T* __restrict__ b) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f < n) b[f] = a[f2d[f]];
}
template <class T>
__global__ void scatter_kernel(int64_t n, const int32_t* __restrict__ f2d, const T* __restrict__ a,
                               T* __restrict__ b) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f < n) b[f2d[f]] = a[f];
}

template <class T>
void gather_free(const Grid& g, const T* node_vec, T* free_vec, cudaStream_t s) {
  if (!g.n_free) return;
  gather_kernel<T><<<grid_blocks(g.n_free, 256), 256, 0, s>>>(g.n_free, g.free2dof.p, node_vec,
                                                              free_vec);
  SG_CHECK_LAUNCH();
}
template <class T>
void scatter_free(const Grid& g, const T* free_vec, T* node_vec, cudaStream_t s) {
  SG_CUDA(cudaMemsetAsync(node_vec, 0, sizeof(T) * 3 * g.d.nnodes(), s));
  if (!g.n_free) return;
  scatter_kernel<T><<<grid_blocks(g.n_free, 256), 256, 0, s>>>(g.n_free, g.free2dof.p, free_vec,
                                                               node_vec);
  SG_CHECK_LAUNCH();
}
template void gather_free<double>(const Grid&, const double*, double*, cudaStream_t);
template void gather_free<float>(const Grid&, const float*, float*, cudaStream_t);
template void scatter_free<double>(const Grid&, const double*, double*, cudaStream_t);
template void scatter_free<float>(const Grid&, const float*, float*, cudaStream_t);

__global__ void f64_to_f32_kernel(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = __double2float_rn(a[i]);
}
__global__ void f32_to_f64_kernel(int64_t n, const float* __restrict__ a, double* __restrict__ b) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = double(a[i]);
}
void cvt_f64_to_f32(int64_t n, const double* a, float* b, cudaStream_t s) {
  if (!n) return;
  f64_to_f32_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(n, a, b);
  SG_CHECK_LAUNCH();
}
void cvt_f32_to_f64(int64_t n, const float* a, double* b, cudaStream_t s) {
  if (!n) return;
  f32_to_f64_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(n, a, b);
  SG_CHECK_LAUNCH();
}

// --------------------------------------------- numpy pairwise summation
// numpy's float64 add.reduce on a contiguous array: blocks of <= 128 summed
// with 8 strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// plus a sequential tail (n < 8: plain loop); longer ranges split at
// n/2 rounded down to a multiple of 8.  We compute the leaves in parallel and
// replay the recursion as a postfix program on one thread.
static void pw_plan(int64_t start, int64_t n, std::vector<int64_t>& leaves,
                    std::vector<uint8_t>& prog) {
  if (n <= 128) {
    leaves.push_back(start);
    leaves.push_back(n);
    prog.push_back(0);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_plan(start, n2, leaves, prog);
  pw_plan(start + n2, n - n2, leaves, prog);
  prog.push_back(1);
}

__global__ void pw_leaf_kernel(int64_t nleaf, const int64_t* __restrict__ leaves,
                               const int32_t* __restrict__ f2d, const double* __restrict__ v,
                               double* __restrict__ out) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L >= nleaf) return;
  const int64_t st = leaves[2 * L], n = leaves[2 * L + 1];
  auto at = [&](int64_t q) { return v[f2d[st + q]]; };
  double res;
  if (n < 8) {
    res = 0.0;
    for (int64_t q = 0; q < n; ++q) res = __dadd_rn(res, at(q));
  } else {
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = at(q);
    int64_t q = 8;
    for (; q < n - (n % 8); q += 8)
      for (int t = 0; t < 8; ++t) r[t] = __dadd_rn(r[t], at(q + t));
    res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; q < n; ++q) res = __dadd_rn(res, at(q));
  }
  out[L] = res;
}

__global__ void pw_combine_kernel(int64_t nprog, const uint8_t* __restrict__ prog,
                                  const double* __restrict__ leafsum, double count,
                                  double* __restrict__ out) {
  double stack[64];
  int sp = 0;
  int64_t next = 0;
  for (int64_t q = 0; q < nprog; ++q) {
    if (prog[q] == 0) {
      stack[sp++] = leafsum[next++];
    } else {
      const double b = stack[--sp];
      const double a = stack[--sp];
      stack[sp++] = __dadd_rn(a, b);
    }
  }
  *out = __ddiv_rn(sp ? stack[0] : 0.0, count);
}

void np_mean_free(const Grid& g, const double* node_vec, double* out_dev, cudaStream_t s) {
  std::vector<int64_t> leaves;
  std::vector<uint8_t> prog;
  pw_plan(0, g.n_free, leaves, prog);
  const int64_t nleaf = int64_t(leaves.size() / 2);
  DBuf<int64_t> dl(leaves.size());
  DBuf<uint8_t> dp(prog.size());
  DBuf<double> ls{size_t(nleaf)};
  dl.upload(leaves.data(), leaves.size(), s);
  dp.upload(prog.data(), prog.size(), s);
  pw_leaf_kernel<<<grid_blocks(nleaf, 128), 128, 0, s>>>(nleaf, dl.p, g.free2dof.p, node_vec, ls.p);
  SG_CHECK_LAUNCH();
  pw_combine_kernel<<<1, 1, 0, s>>>(int64_t(prog.size()), dp.p, ls.p, double(g.n_free), out_dev);
  SG_CHECK_LAUNCH();
  SG_CUDA(cudaStreamSynchronize(s));  // temporaries die here
}

__global__ void diag_floor_kernel(int64_t n, const int32_t* __restrict__ f2d, double* __restrict__ d,
                                  const double* __restrict__ mean) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const double fl = __dmul_rn(1e-14, *mean);
  const int32_t q = f2d[f];
  d[q] = fmax(d[q], fl);
}
void diag_floor(const Grid& g, double* d, const double* mean_dev, cudaStream_t s) {
  if (!g.n_free) return;
  diag_floor_kernel<<<grid_blocks(g.n_free, 256), 256, 0, s>>>(g.n_free, g.free2dof.p, d, mean_dev);
  SG_CHECK_LAUNCH();
}

// ------------------------------------------------ seeded gaussian vectors
// SplitMix64(seed).gaussian(n) in free order (prng.py:26-64): output t uses
// counters t+1 (u1) and m+t+1 (u2), m = ceil(n/2); Box-Muller pairs.
__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * ctr;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gauss_kernel(int64_t n, uint64_t seed, const int32_t* __restrict__ f2d,
                             double* __restrict__ v) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int64_t m = (n + 1) / 2;
  const int64_t t = f / 2;
  const double u1 = (double(splitmix(seed, uint64_t(t + 1)) >> 11) + 1.0) * 0x1p-53;
  const double u2 = double(splitmix(seed, uint64_t(m + t + 1)) >> 11) * 0x1p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.141592653589793 * u2;
  v[f2d[f]] = (f & 1) ? r * sin(th) : r * cos(th);
}

struct SqNorm {
  const double* v;
  __device__ void operator()(int64_t i, double (&acc)[1]) const { acc[0] += v[i] * v[i]; }
};
__global__ void scale_by_inv_sqrt(int64_t n, double* v, const double* ss) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double nrm = sqrt(*ss);
  if (nrm != 0.0) v[i] = v[i] / nrm;
}

void fill_gaussian_unit(const Grid& g, uint64_t seed, double* v, RedWork& w, double* scratch,
                        cudaStream_t s) {
  const int64_t nd = 3 * g.d.nnodes();
  SG_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * nd, s));
  if (!g.n_free) return;
  gauss_kernel<<<grid_blocks(g.n_free, 256), 256, 0, s>>>(g.n_free, seed, g.free2dof.p, v);
  SG_CHECK_LAUNCH();
  launch_reduce<1>(nd, SqNorm{v}, StoreTo<1>{{scratch}}, w, s);
  scale_by_inv_sqrt<<<grid_blocks(nd, 256), 256, 0, s>>>(nd, v, scratch);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
