// Structured trilinear prolongation / restriction (transfer.py:42-107).
//
// P is never stored: weights {1, 1/2} per axis are recomputed from node
// parity.  Products with dyadic weights are exact and the sums follow the
// reference's order (csr_matvec: ascending coarse column for P x;
// csc_matvec of P^T: ascending fine row for P^T x) with FMA-free adds, so
// both transfers are bit-identical to the scipy reference.
#include <algorithm>
#include "sg_kernels.cuh"

namespace sg {

__global__ void prolong_kernel(GridDesc f, GridDesc c, const uint8_t* __restrict__ fmask,
                               const uint8_t* __restrict__ cmask, const double* __restrict__ xc,
                               double* __restrict__ xf, bool add, float* __restrict__ xp32, int XS) {
  const int64_t nn = f.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int FX = f.nx + 1, FY = f.ny + 1, CX = c.nx + 1, CY = c.ny + 1;
  const int nd32 = int(node), jk = nd32 / FX;  // 32-bit index math
  const int i = nd32 - jk * FX, j = jk % FY, k = jk / FY;
  int pi[2], pj[2], pk[2];
  double wi, wj, wk;
  int ni, nj, nk;
  if (i & 1) { pi[0] = i >> 1; pi[1] = (i >> 1) + 1; ni = 2; wi = 0.5; } else { pi[0] = i >> 1; ni = 1; wi = 1.0; }
  if (j & 1) { pj[0] = j >> 1; pj[1] = (j >> 1) + 1; nj = 2; wj = 0.5; } else { pj[0] = j >> 1; nj = 1; wj = 1.0; }
  if (k & 1) { pk[0] = k >> 1; pk[1] = (k >> 1) + 1; nk = 2; wk = 0.5; } else { pk[0] = k >> 1; nk = 1; wk = 1.0; }
  const double w = wi * wj * wk;  // exact dyadic
  double s[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nj; ++b)
      for (int q = 0; q < ni; ++q) {
        const int64_t cn = pi[q] + int64_t(CX) * (pj[b] + int64_t(CY) * pk[a]);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          if (!node_fixed_axis(c, cmask, cn, pi[q], ax))
            s[ax] = __dadd_rn(s[ax], __dmul_rn(w, xc[3 * cn + ax]));
      }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    float* o32 = xp32 ? xp32 + ((int64_t(k) * FY + j) * 3 + ax) * XS + i : nullptr;
    if (!xf) {
      // V-cycle on a P32 level: the f64 iterate is f64(x32) exactly, so the
      // sum is formed from the P32 copy and only f32(x + P e) is stored
      const double base = double(*o32);
      const double v = node_fixed_axis(f, fmask, node, i, ax) ? base : __dadd_rn(base, s[ax]);
      *o32 = __double2float_rn(v);
      continue;
    }
    double* o = xf + 3 * node + ax;
    double v;
    if (node_fixed_axis(f, fmask, node, i, ax)) {
      v = add ? *o : 0.0;
      if (!add) *o = 0.0;
    } else {
      v = add ? __dadd_rn(*o, s[ax]) : s[ax];
      *o = v;
    }
    // level-0 P32 copy f32(x) for the post-smoother (sg_fine_pk.cu layout)
    if (o32) *o32 = __double2float_rn(v);
  }
}

__global__ void restrict_kernel(GridDesc f, GridDesc c, const uint8_t* __restrict__ fmask,
                                const uint8_t* __restrict__ cmask, const double* __restrict__ xf,
                                double* __restrict__ xc) {
  const int64_t nn = c.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int FX = f.nx + 1, FY = f.ny + 1, CX = c.nx + 1, CY = c.ny + 1;
  const int nd32 = int(node), jk = nd32 / CX;  // 32-bit index math
  const int i = nd32 - jk * CX, j = jk % CY, k = jk / CY;
  double s[3] = {0.0, 0.0, 0.0};
  for (int dk = -1; dk <= 1; ++dk) {
    const int fk = 2 * k + dk;
    if (fk < 0 || fk > f.nz) continue;
    const double wk = dk ? 0.5 : 1.0;
    for (int dj = -1; dj <= 1; ++dj) {
      const int fj = 2 * j + dj;
      if (fj < 0 || fj > f.ny) continue;
      const double wj = dj ? 0.5 : 1.0;
      for (int di = -1; di <= 1; ++di) {
        const int fi = 2 * i + di;
        if (fi < 0 || fi > f.nx) continue;
        const double w = (di ? 0.5 : 1.0) * wj * wk;
        const int64_t fn = fi + int64_t(FX) * (fj + int64_t(FY) * fk);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          if (!node_fixed_axis(f, fmask, fn, fi, ax))
            s[ax] = __dadd_rn(s[ax], __dmul_rn(w, xf[3 * fn + ax]));
      }
    }
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax)
    xc[3 * node + ax] = node_fixed_axis(c, cmask, node, i, ax) ? 0.0 : s[ax];
}

void prolong(const Grid& fine, const Grid& coarse, const double* xc, double* xf, bool add,
             cudaStream_t s, float* xp32, int XS) {
  const int64_t nn = fine.d.nnodes();
  prolong_kernel<<<grid_blocks(nn, 256), 256, 0, s>>>(fine.d, coarse.d, fine.nmask.p,
                                                      coarse.nmask.p, xc, xf, add, xp32, XS);
  SG_CHECK_LAUNCH();
}

void restrict_(const Grid& fine, const Grid& coarse, const double* xf, double* xc,
               cudaStream_t s) {
  const int64_t nn = coarse.d.nnodes();
  restrict_kernel<<<grid_blocks(nn, 256), 256, 0, s>>>(fine.d, coarse.d, fine.nmask.p,
                                                       coarse.nmask.p, xf, xc);
  SG_CHECK_LAUNCH();
}

// P in canonical CSR (transfer.py:85-107) for inspection / parity checks.
__global__ void p_rows_kernel(GridDesc f, GridDesc c, int64_t nfree, const int32_t* __restrict__ f2d,
                              const int32_t* __restrict__ cd2f, const int64_t* __restrict__ indptr,
                              int64_t* __restrict__ counts, int64_t* __restrict__ indices,
                              double* __restrict__ data) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nfree) return;
  const int FX = f.nx + 1, FY = f.ny + 1, CX = c.nx + 1, CY = c.ny + 1;
  const int64_t node = f2d[r] / 3;
  const int ax = f2d[r] % 3;
  const int nd32 = int(node), jk = nd32 / FX;  // 32-bit index math
  const int i = nd32 - jk * FX, j = jk % FY, k = jk / FY;
  const int ni = (i & 1) ? 2 : 1, nj = (j & 1) ? 2 : 1, nk = (k & 1) ? 2 : 1;
  const double w = ((i & 1) ? 0.5 : 1.0) * ((j & 1) ? 0.5 : 1.0) * ((k & 1) ? 0.5 : 1.0);
  int64_t o = indptr ? indptr[r] : 0, cnt = 0;
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nj; ++b)
      for (int q = 0; q < ni; ++q) {
        const int64_t cn = ((i >> 1) + q) + int64_t(CX) * (((j >> 1) + b) + int64_t(CY) * ((k >> 1) + a));
        const int32_t col = cd2f[3 * cn + ax];
        if (col < 0) continue;
        if (indices) {
          indices[o] = col;
          data[o] = w;
          ++o;
        }
        ++cnt;
      }
  if (counts) counts[r] = cnt;
}

void transfer_export_csr(const Grid& fine, const Grid& coarse, int64_t* indptr_h, int64_t* indices_h,
                         double* data_h, int64_t* nnz_out, cudaStream_t s) {
  const int64_t nf = fine.n_free;
  DBuf<int64_t> cnt(static_cast<size_t>(std::max<int64_t>(nf, 1)));
  if (nf)
    p_rows_kernel<<<grid_blocks(nf, 128), 128, 0, s>>>(fine.d, coarse.d, nf, fine.free2dof.p,
                                                       coarse.dof2free.p, nullptr, cnt.p, nullptr, nullptr);
  SG_CHECK_LAUNCH();
  std::vector<int64_t> h(static_cast<size_t>(nf)), ptr(static_cast<size_t>(nf + 1), 0);
  cnt.download(h.data(), size_t(nf), s);
  SG_CUDA(cudaStreamSynchronize(s));
  for (int64_t r = 0; r < nf; ++r) ptr[size_t(r + 1)] = ptr[size_t(r)] + h[size_t(r)];
  *nnz_out = ptr.back();
  if (!indices_h) return;
  const int64_t nnz = ptr.back();
  DBuf<int64_t> dptr(ptr.size()), dind(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  DBuf<double> ddat(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  dptr.upload(ptr.data(), ptr.size(), s);
  if (nf)
    p_rows_kernel<<<grid_blocks(nf, 128), 128, 0, s>>>(fine.d, coarse.d, nf, fine.free2dof.p,
                                                       coarse.dof2free.p, dptr.p, nullptr, dind.p, ddat.p);
  SG_CHECK_LAUNCH();
  dind.download(indices_h, size_t(nnz), s);
  ddat.download(data_h, size_t(nnz), s);
  SG_CUDA(cudaStreamSynchronize(s));
  std::copy(ptr.begin(), ptr.end(), indptr_h);
}

}  // namespace sg
