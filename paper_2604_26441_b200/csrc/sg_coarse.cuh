#pragma once
#include "sg_kernels.cuh"

namespace sg {

// Fixed-count Jacobi-PCG on K + eps I (hierarchy.py:139-162), one
// persistent cooperative launch per solve.
struct Pcg80 {
  const Grid* grid = nullptr;
  const double* Aptr = nullptr;
  double eps = 0.0;
  int steps = 80;
  int nblocks = 0;
  int cache_slots = 0; // stencil slots resident in shared memory
  int smem_bytes = 0;
  DBuf<double> dinv, r, z, p0, p1, q, partials;
  DBuf<unsigned> bar;
  // brick-partitioned kernel (pcg80_brick_kernel) when the level fits on chip
  bool brick = false;
  int variant = 2;  // 0 Hestenes-Stiefel, 1 Chronopoulos-Gear, 2 pipelined (sg_coarse.cu)
  int sx = 0, sy = 0, sz = 0;
  int nrep = 1, poll_ns = 0;  // variant 3 all-reduce tuning (sg_coarse.cu)
  DBuf<uint4> slots, zll;
  DBuf<double> apk;  // operator packed per brick (pipelined variants)
  DBuf<unsigned long long> bstate;
  void setup(const Grid& g, const double* A, const double* diag, double eps, int steps,
             cudaStream_t s);
  void solve(const double* b, double* x, cudaStream_t s);
  long long* trace = nullptr;  // development instrumentation (sg_hier_pcg80_trace)
};

// Brick split of a coarsest grid for the pcg80 brick kernel (host only):
// sx*sy*sz <= nsm bricks of <= 144 nodes, halo window <= 448 nodes.
bool brick_plan(const GridDesc& g, int nsm, int& sx, int& sy, int& sz);

// Blocked device Cholesky + explicit inverse of an SPD n x n row-major matrix
// (sg_dense.cu); returns false on a non-positive pivot.
bool dense_spd_inverse(int n, double* A, double* Ainv, cudaStream_t s);

// Dense (K + eps I)^-1 from an on-device Cholesky (hierarchy.py:165-178).
struct DenseInverse {
  const Grid* grid = nullptr;
  int64_t n = 0;
  DBuf<double> Ainv;  // n x n, free ordering
  bool setup(const Grid& g, const double* dense_with_eps, cudaStream_t s);
  void solve(const double* r, double* x, cudaStream_t s);
};

}  // namespace sg
