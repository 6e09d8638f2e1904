// Level-0 matrix-free operator: y = K_ff u for a rho^p-scaled Q1 element
// stiffness on a structured hexahedral grid (reference: FineOperator.matvec_tagged,
// fine_operator.py:56-77; diagonal fine_operator.py:79-86).
//
// Output-stationary (node-centric) formulation: each node sums the
// contributions of its <= 8 adjacent elements in ascending element order, so
// no atomics are needed and every result is bit-reproducible run to run.
// The modulus is applied after the element contraction, as in the reference.
#include <cstdlib>
#include "sg_kernels.cuh"

namespace sg {

template <class T, int TAG>
__global__ void __launch_bounds__(256) fine_apply_kernel(GridDesc g, const uint8_t* __restrict__ nmask,
                                                         const T* __restrict__ u, T* __restrict__ y,
                                                         const T* __restrict__ E, KeParam<T> ke) {
  const int64_t nn = g.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int i = int(node % NX);
  const int j = int((node / NX) % NY);
  const int k = int(node / (int64_t(NX) * NY));
  T acc0 = 0, acc1 = 0, acc2 = 0;
  for (int dk = -1; dk <= 0; ++dk) {
    const int ek = k + dk;
    if (ek < 0 || ek >= g.nz) continue;
    for (int dj = -1; dj <= 0; ++dj) {
      const int ej = j + dj;
      if (ej < 0 || ej >= g.ny) continue;
      for (int di = -1; di <= 0; ++di) {
        const int ei = i + di;
        if (ei < 0 || ei >= g.nx) continue;
        const int64_t e = ei + int64_t(g.nx) * (ej + int64_t(g.ny) * ek);
        const int a = -di + 2 * (-dj) + 4 * (-dk);
        T l0 = 0, l1 = 0, l2 = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int64_t nb = (ei + (b & 1)) + int64_t(NX) * ((ej + ((b >> 1) & 1)) + int64_t(NY) * (ek + (b >> 2)));
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            T uv = u[3 * nb + c];
            if (TAG == 2) uv = bf16_round(uv);
            const int col = 3 * b + c;
            l0 += ke.k[(3 * a + 0) * 24 + col] * uv;
            l1 += ke.k[(3 * a + 1) * 24 + col] * uv;
            l2 += ke.k[(3 * a + 2) * 24 + col] * uv;
          }
        }
        const T ev = E[e];
        acc0 += l0 * ev;
        acc1 += l1 * ev;
        acc2 += l2 * ev;
      }
    }
  }
  T* yo = y + 3 * node;
  yo[0] = node_fixed_axis(g, nmask, node, i, 0) ? T(0) : acc0;
  yo[1] = node_fixed_axis(g, nmask, node, i, 1) ? T(0) : acc1;
  yo[2] = node_fixed_axis(g, nmask, node, i, 2) ? T(0) : acc2;
}

// diag(K_ff) in ascending element order with FMA-free FP64: bit-identical to
// np.bincount(edofs, E*diag(ke)) (fine_operator.py:82-85).
__global__ void fine_diag_kernel(GridDesc g, const uint8_t* __restrict__ nmask,
                                 const double* __restrict__ E, KeDiag kd, double* __restrict__ d) {
  const int64_t nn = g.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int i = int(node % NX);
  const int j = int((node / NX) % NY);
  const int k = int(node / (int64_t(NX) * NY));
  double acc[3] = {0.0, 0.0, 0.0};
  for (int dk = -1; dk <= 0; ++dk) {
    const int ek = k + dk;
    if (ek < 0 || ek >= g.nz) continue;
    for (int dj = -1; dj <= 0; ++dj) {
      const int ej = j + dj;
      if (ej < 0 || ej >= g.ny) continue;
      for (int di = -1; di <= 0; ++di) {
        const int ei = i + di;
        if (ei < 0 || ei >= g.nx) continue;
        const int64_t e = ei + int64_t(g.nx) * (ej + int64_t(g.ny) * ek);
        const int a = -di - 2 * dj - 4 * dk;
        const double ev = E[e];
#pragma unroll
        for (int r = 0; r < 3; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(ev, kd.d[3 * a + r]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) d[3 * node + r] = node_fixed_axis(g, nmask, node, i, r) ? 0.0 : acc[r];
}

template <class T, int TAG>
static void launch_apply(const GridDesc& g, const uint8_t* nmask, const T* u, T* y, const T* E,
                         const KeParam<T>& ke, cudaStream_t s) {
  const int64_t nn = g.nnodes();
  fine_apply_kernel<T, TAG><<<grid_blocks(nn, 256), 256, 0, s>>>(g, nmask, u, y, E, ke);
  SG_CHECK_LAUNCH();
}

void fine_apply_dense_f64(const FineOp& op, const double* u, double* y, cudaStream_t s) {
  launch_apply<double, 0>(op.grid.d, op.grid.nmask.p, u, y, op.E64.p, op.ke64, s);
}
void fine_apply_dense_f32(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  launch_apply<float, 1>(op.grid.d, op.grid.nmask.p, u, y, op.E32.p, op.ke32, s);
}
// FP64: the block-form Walsh kernel with plane-shared transforms
// (sg_fine_p64.cu); SG_WALSH64_OLD=1 selects the scalar full-Walsh kernel.
void fine_apply_f64(const FineOp& op, const double* u, double* y, cudaStream_t s) {
  static const bool old = getenv("SG_WALSH64_OLD") != nullptr;
  if (!old && p64_supported(op)) fine_apply_p64(op, u, y, s);
  else if (op.walsh_ok) fine_apply_walsh_f64(op, u, y, s);
  else fine_apply_dense_f64(op, u, y, s);
}
// FP32 on node-layout vectors: converted through the P32 layout and the
// packed FP32x2 kernel (sg_fine_pk.cu); SG_FINE_WALSH1=1 selects the scalar
// one-element-per-thread Walsh kernel (comparison runs).
void fine_apply_f32(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  static const bool scalar = getenv("SG_FINE_WALSH1") != nullptr;
  if (!scalar && op.p32a.n >= size_t(p32_size(op.grid.d)) && p32_supported(op)) {
    FineOp& m = const_cast<FineOp&>(op);
    to_p32<float>(op.grid.d, u, m.p32a.p, s);
    fine_apply_p32(op, m.p32a.p, m.p32b.p, s);
    from_p32<float>(op.grid.d, m.p32b.p, y, s);
    return;
  }
  if (op.walsh_ok) fine_apply_walsh_f32(op, u, y, s);
  else fine_apply_dense_f32(op, u, y, s);
}
void fine_apply_bf16_dense(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  launch_apply<float, 2>(op.grid.d, op.grid.nmask.p, u, y, op.E32.p, op.ke16, s);
}
// BF16EMU runs on the tensor cores: the record-fed pipelined kernel
// (sg_fine_tc2.cu), or for grids wider than it supports the per-element one
// (sg_fine_tc.cu, also SG_BF16_TC1=1); SG_BF16_DENSE=1 selects the CUDA-core
// reference kernel (used by the parity tests).
void fine_apply_bf16(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  static const bool dense = [] {
    const char* e = std::getenv("SG_BF16_DENSE");
    return e && e[0] == '1';
  }();
  static const bool tc1 = std::getenv("SG_BF16_TC1") != nullptr;  // per-element staging kernel
  if (dense) fine_apply_bf16_dense(op, u, y, s);
  else if (tc1 || !fine_apply_bf16_tc2(op, u, y, s)) fine_apply_bf16_tc(op, u, y, s);
}

void fine_diag_raw(const FineOp& op, double* d, cudaStream_t s) {
  const int64_t nn = op.grid.d.nnodes();
  fine_diag_kernel<<<grid_blocks(nn, 256), 256, 0, s>>>(op.grid.d, op.grid.nmask.p, op.E64.p,
                                                         op.kdiag, d);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
