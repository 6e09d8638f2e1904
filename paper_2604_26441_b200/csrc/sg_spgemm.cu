// General CSR sparse triple product P^T (K P) with scipy's summation order
// (transfer.py:177-181 on arbitrary CSR inputs; the structured hierarchy uses
// the stencil kernels of sg_galerkin.cu instead).
//
// scipy evaluates K @ P with csr_matmat: for row j the terms of entry (j,k)
// are accumulated sequentially in (stored entry of K row j, stored entry of P
// row m) order, exact zeros dropped.  P.T @ KP runs as csc_matmat, i.e. entry
// (i,k) sums KP[j,k] * P[j,i] over ascending j.  Both are the same row-wise
// Gustavson product: C = A B with each output row accumulated by ONE thread in
// the stored order of A's row and B's rows, so the device result is
// bit-identical.  (Index bookkeeping -- prefix sums and the stable transpose
// of P -- is host C++.)
#include <algorithm>
#include "sg_kernels.cuh"

namespace sg {

__global__ void matmat_ub_kernel(int64_t n_row, const int64_t* __restrict__ Ap,
                                 const int64_t* __restrict__ Aj, const int64_t* __restrict__ Bp,
                                 int64_t* __restrict__ ub) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_row) return;
  int64_t s = 0;
  for (int64_t jj = Ap[i]; jj < Ap[i + 1]; ++jj) s += Bp[Aj[jj] + 1] - Bp[Aj[jj]];
  ub[i] = s;
}

// Row-wise numeric product with an open-addressing hash per row (capacity a
// power of two >= 2*ub).  keys/vals hold the hash; order[] the first-touch order.
__global__ void matmat_num_kernel(int64_t n_row, const int64_t* __restrict__ Ap,
                                  const int64_t* __restrict__ Aj, const double* __restrict__ Ax,
                                  const int64_t* __restrict__ Bp, const int64_t* __restrict__ Bj,
                                  const double* __restrict__ Bx, const int64_t* __restrict__ hoff,
                                  int64_t* __restrict__ keys, double* __restrict__ vals,
                                  const int64_t* __restrict__ ooff, int64_t* __restrict__ order,
                                  int64_t* __restrict__ cnt) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_row) return;
  const int64_t h0 = hoff[i], cap = hoff[i + 1] - hoff[i];
  int64_t* K = keys + h0;
  double* V = vals + h0;
  int64_t* O = order + ooff[i];
  for (int64_t q = 0; q < cap; ++q) K[q] = -1;
  int64_t n = 0;
  for (int64_t jj = Ap[i]; jj < Ap[i + 1]; ++jj) {
    const int64_t j = Aj[jj];
    const double v = Ax[jj];
    for (int64_t kk = Bp[j]; kk < Bp[j + 1]; ++kk) {
      const int64_t k = Bj[kk];
      const double t = __dmul_rn(v, Bx[kk]);
      int64_t h = (k * 0x9E3779B97F4A7C15ull >> 17) & (cap - 1);
      while (K[h] != -1 && K[h] != k) h = (h + 1) & (cap - 1);
      if (K[h] == -1) {
        K[h] = k;
        V[h] = __dadd_rn(0.0, t);  // scipy: sums[k] starts at 0
        O[n++] = h;
      } else {
        V[h] = __dadd_rn(V[h], t);
      }
    }
  }
  cnt[i] = n;
}

// Compact: nonzero sums, columns sorted ascending (insertion sort, short rows).
__global__ void matmat_out_kernel(int64_t n_row, const int64_t* __restrict__ hoff,
                                  const int64_t* __restrict__ keys, const double* __restrict__ vals,
                                  const int64_t* __restrict__ ooff, const int64_t* __restrict__ order,
                                  const int64_t* __restrict__ cnt, const int64_t* __restrict__ Cp,
                                  int64_t* __restrict__ Cj, double* __restrict__ Cx, bool count_only,
                                  int64_t* __restrict__ nz) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_row) return;
  const int64_t* K = keys + hoff[i];
  const double* V = vals + hoff[i];
  const int64_t* O = order + ooff[i];
  if (count_only) {
    int64_t c = 0;
    for (int64_t q = 0; q < cnt[i]; ++q) c += V[O[q]] != 0.0;
    nz[i] = c;
    return;
  }
  int64_t o = Cp[i];
  const int64_t start = o;
  for (int64_t q = 0; q < cnt[i]; ++q) {
    const double v = V[O[q]];
    if (v == 0.0) continue;
    const int64_t k = K[O[q]];
    int64_t p = o++;
    while (p > start && Cj[p - 1] > k) {
      Cj[p] = Cj[p - 1];
      Cx[p] = Cx[p - 1];
      --p;
    }
    Cj[p] = k;
    Cx[p] = v;
  }
}

struct HostCsr {
  int64_t nr = 0, nc = 0;
  std::vector<int64_t> p, j;
  std::vector<double> x;
};

// C = A @ B (scipy csr_matmat semantics) on the device.
static HostCsr device_matmat(const HostCsr& A, const HostCsr& B, cudaStream_t s) {
  const int64_t n = A.nr;
  HostCsr C;
  C.nr = n;
  C.nc = B.nc;
  C.p.assign(size_t(n + 1), 0);
  if (n == 0) return C;
  DBuf<int64_t> dAp(A.p.size()), dAj(std::max<size_t>(A.j.size(), 1)), dBp(B.p.size()),
      dBj(std::max<size_t>(B.j.size(), 1)), ub(static_cast<size_t>(n));
  DBuf<double> dAx(std::max<size_t>(A.x.size(), 1)), dBx(std::max<size_t>(B.x.size(), 1));
  dAp.upload(A.p.data(), A.p.size(), s);
  dAj.upload(A.j.data(), A.j.size(), s);
  dAx.upload(A.x.data(), A.x.size(), s);
  dBp.upload(B.p.data(), B.p.size(), s);
  dBj.upload(B.j.data(), B.j.size(), s);
  dBx.upload(B.x.data(), B.x.size(), s);
  const int nb = grid_blocks(n, 128);
  matmat_ub_kernel<<<nb, 128, 0, s>>>(n, dAp.p, dAj.p, dBp.p, ub.p);
  SG_CHECK_LAUNCH();
  std::vector<int64_t> hub(static_cast<size_t>(n));
  ub.download(hub.data(), hub.size(), s);
  SG_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> hoff(size_t(n + 1), 0), ooff(size_t(n + 1), 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t cap = 1;
    while (cap < 2 * hub[size_t(i)]) cap <<= 1;
    hoff[size_t(i + 1)] = hoff[size_t(i)] + cap;
    ooff[size_t(i + 1)] = ooff[size_t(i)] + hub[size_t(i)];
  }
  DBuf<int64_t> dh(hoff.size()), doo(ooff.size()), keys(static_cast<size_t>(std::max<int64_t>(hoff.back(), 1))),
      order(static_cast<size_t>(std::max<int64_t>(ooff.back(), 1))), cnt(static_cast<size_t>(n)),
      nz(static_cast<size_t>(n));
  DBuf<double> vals(static_cast<size_t>(std::max<int64_t>(hoff.back(), 1)));
  dh.upload(hoff.data(), hoff.size(), s);
  doo.upload(ooff.data(), ooff.size(), s);
  matmat_num_kernel<<<nb, 128, 0, s>>>(n, dAp.p, dAj.p, dAx.p, dBp.p, dBj.p, dBx.p, dh.p, keys.p,
                                       vals.p, doo.p, order.p, cnt.p);
  SG_CHECK_LAUNCH();
  matmat_out_kernel<<<nb, 128, 0, s>>>(n, dh.p, keys.p, vals.p, doo.p, order.p, cnt.p, nullptr,
                                       nullptr, nullptr, true, nz.p);
  SG_CHECK_LAUNCH();
  std::vector<int64_t> hnz(static_cast<size_t>(n));
  nz.download(hnz.data(), hnz.size(), s);
  SG_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) C.p[size_t(i + 1)] = C.p[size_t(i)] + hnz[size_t(i)];
  const int64_t nnz = C.p.back();
  C.j.assign(size_t(nnz), 0);
  C.x.assign(size_t(nnz), 0.0);
  if (nnz) {
    DBuf<int64_t> dCp(C.p.size()), dCj(static_cast<size_t>(nnz));
    DBuf<double> dCx(static_cast<size_t>(nnz));
    dCp.upload(C.p.data(), C.p.size(), s);
    matmat_out_kernel<<<nb, 128, 0, s>>>(n, dh.p, keys.p, vals.p, doo.p, order.p, cnt.p, dCp.p,
                                         dCj.p, dCx.p, false, nullptr);
    SG_CHECK_LAUNCH();
    dCj.download(C.j.data(), size_t(nnz), s);
    dCx.download(C.x.data(), size_t(nnz), s);
    SG_CUDA(cudaStreamSynchronize(s));
  }
  return C;
}

// Stable transpose (csr_tocsc semantics: row indices ascending per column).
static HostCsr transpose(const HostCsr& A) {
  HostCsr T;
  T.nr = A.nc;
  T.nc = A.nr;
  T.p.assign(size_t(A.nc + 1), 0);
  for (int64_t q = 0; q < int64_t(A.j.size()); ++q) T.p[size_t(A.j[size_t(q)] + 1)]++;
  for (int64_t c = 0; c < A.nc; ++c) T.p[size_t(c + 1)] += T.p[size_t(c)];
  std::vector<int64_t> next(T.p.begin(), T.p.end() - 1);
  T.j.assign(A.j.size(), 0);
  T.x.assign(A.x.size(), 0.0);
  for (int64_t r = 0; r < A.nr; ++r)
    for (int64_t q = A.p[size_t(r)]; q < A.p[size_t(r + 1)]; ++q) {
      const int64_t d = next[size_t(A.j[size_t(q)])]++;
      T.j[size_t(d)] = r;
      T.x[size_t(d)] = A.x[size_t(q)];
    }
  return T;
}

struct PtapResult {
  HostCsr C;
};

void* ptap_compute(int64_t nf, int64_t nc, const int64_t* Pp, const int64_t* Pj, const double* Px,
                   const int64_t* Kp, const int64_t* Kj, const double* Kx, int64_t* nnz,
                   cudaStream_t s) {
  HostCsr P, K;
  P.nr = nf;
  P.nc = nc;
  P.p.assign(Pp, Pp + nf + 1);
  P.j.assign(Pj, Pj + P.p.back());
  P.x.assign(Px, Px + P.p.back());
  K.nr = nf;
  K.nc = nf;
  K.p.assign(Kp, Kp + nf + 1);
  K.j.assign(Kj, Kj + K.p.back());
  K.x.assign(Kx, Kx + K.p.back());
  HostCsr KP = device_matmat(K, P, s);   // K @ P
  HostCsr PT = transpose(P);             // P^T as CSR, j ascending per row
  auto* R = new PtapResult;
  R->C = device_matmat(PT, KP, s);       // P^T @ KP, sums over ascending j
  *nnz = R->C.p.back();
  return R;
}

void ptap_fetch(void* h, int64_t* Cp, int64_t* Cj, double* Cx) {
  auto* R = static_cast<PtapResult*>(h);
  std::copy(R->C.p.begin(), R->C.p.end(), Cp);
  std::copy(R->C.j.begin(), R->C.j.end(), Cj);
  std::copy(R->C.x.begin(), R->C.x.end(), Cx);
}

void ptap_free(void* h) { delete static_cast<PtapResult*>(h); }

}  // namespace sg
