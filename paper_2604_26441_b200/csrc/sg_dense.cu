// Dense coarsest solve (hierarchy.py:165-178): blocked right-looking Cholesky of
// K + eps I on the device (64-wide panels: one-CTA panel factorisation,
// row-parallel triangular solve, tiled FP64 GEMM trailing update), then the
// explicit inverse (L^-1 by blocked forward substitution, A^-1 = L^-T L^-1),
// so that every V-cycle's coarsest solve is a single GEMV.  Setup-only work;
// a non-positive pivot reports failure and the hierarchy falls back to pcg80
// exactly like the reference's LinAlgError branch.
#include <cmath>
#include "sg_coarse.cuh"

namespace sg {

constexpr int kNB = 64;  // panel width

// C(i,j) = beta * C(i,j) + alpha * sum_k A(i,k) B(k,j) with arbitrary strides
// (element (i,k) of A at A[i*sai + k*sak], etc.).  64x64 tiles, 256 threads,
// 4x4 outputs per thread, K staged through shared memory 16 at a time.
__global__ void __launch_bounds__(256) gemm_strided_kernel(int M, int N, int K, double alpha,
                                                           const double* __restrict__ A,
                                                           int64_t sai, int64_t sak,
                                                           const double* __restrict__ B,
                                                           int64_t sbk, int64_t sbj, double beta,
                                                           double* __restrict__ C, int64_t sci,
                                                           int64_t scj) {
  __shared__ double As[16][65];
  __shared__ double Bs[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int t = threadIdx.x; t < 16 * 64; t += 256) {
      const int kk = t / 64, r = t % 64;
      const int ia = i0 + r, ka = k0 + kk;
      As[kk][r] = (ia < M && ka < K) ? A[int64_t(ia) * sai + int64_t(ka) * sak] : 0.0;
      const int jb = j0 + r;
      Bs[kk][r] = (jb < N && ka < K) ? B[int64_t(ka) * sbk + int64_t(jb) * sbj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][ty + 16 * q];
        b[q] = Bs[kk][tx + 16 * q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ty + 16 * p, j = j0 + tx + 16 * q;
      if (i < M && j < N) {
        double* c = C + int64_t(i) * sci + int64_t(j) * scj;
        *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * acc[p][q];
      }
    }
}

static void gemm(int M, int N, int K, double alpha, const double* A, int64_t sai, int64_t sak,
                 const double* B, int64_t sbk, int64_t sbj, double beta, double* C, int64_t sci,
                 int64_t scj, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  gemm_strided_kernel<<<grid, 256, 0, s>>>(M, N, K, alpha, A, sai, sak, B, sbk, sbj, beta, C, sci, scj);
  SG_CHECK_LAUNCH();
}

// Unblocked Cholesky of the b x b diagonal block (row-major, ld = n), one CTA.
__global__ void potrf_block_kernel(int n, int j0, int b, double* L, int* info) {
  __shared__ double T[kNB][kNB + 1];
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int r = t / b, c = t % b;
    T[r][c] = L[int64_t(j0 + r) * n + j0 + c];
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      const double d = T[j][j];
      if (!(d > 0.0) || !isfinite(d)) bad = j0 + j + 1;
      else T[j][j] = sqrt(d);
    }
    __syncthreads();
    if (bad) break;
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x) T[i][j] /= T[j][j];
    __syncthreads();
    for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
      const int i = t / b, k = t % b;
      if (i > j && k > j && k <= i) T[i][k] -= T[i][j] * T[k][j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && bad && *info == 0) *info = bad;
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int r = t / b, c = t % b;
    L[int64_t(j0 + r) * n + j0 + c] = c <= r ? T[r][c] : 0.0;
  }
}

// Rows below the panel: L21 = A21 * L11^-T (forward substitution per row).
__global__ void trsm_rows_kernel(int n, int j0, int b, double* L) {
  __shared__ double T[kNB][kNB + 1];
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int r = t / b, c = t % b;
    T[r][c] = L[int64_t(j0 + r) * n + j0 + c];
  }
  __syncthreads();
  const int row = j0 + b + blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double x[kNB];
  double* a = L + int64_t(row) * n + j0;
  for (int c = 0; c < b; ++c) {
    double s = a[c];
    for (int k = 0; k < c; ++k) s -= x[k] * T[c][k];
    x[c] = s / T[c][c];
  }
  for (int c = 0; c < b; ++c) a[c] = x[c];
}

// Block row ib of L^-1: Y = L_ii^-1 * R, R (b x ncols, row-major ld n) in place.
__global__ void trsm_cols_kernel(int n, int i0, int b, int ncols, const double* __restrict__ L,
                                 double* __restrict__ Y) {
  __shared__ double T[kNB][kNB + 1];
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int r = t / b, c = t % b;
    T[r][c] = L[int64_t(i0 + r) * n + i0 + c];
  }
  __syncthreads();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double x[kNB];
  for (int r = 0; r < b; ++r) {
    double s = Y[int64_t(i0 + r) * n + col];
    for (int k = 0; k < r; ++k) s -= T[r][k] * x[k];
    x[r] = s / T[r][r];
  }
  for (int r = 0; r < b; ++r) Y[int64_t(i0 + r) * n + col] = x[r];
}

__global__ void identity_kernel(int n, double* Y) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= int64_t(n) * n) return;
  Y[q] = (q / n == q % n) ? 1.0 : 0.0;
}

// Returns false on a non-positive pivot (dpotrf info > 0).
bool dense_spd_inverse(int n, double* A /* in: SPD, destroyed */, double* Ainv, cudaStream_t s) {
  DBuf<int> info(1);
  info.zero(s);
  for (int j0 = 0; j0 < n; j0 += kNB) {
    const int b = std::min(kNB, n - j0);
    potrf_block_kernel<<<1, 256, 0, s>>>(n, j0, b, A, info.p);
    SG_CHECK_LAUNCH();
    const int rows = n - j0 - b;
    if (rows > 0) {
      trsm_rows_kernel<<<(rows + 127) / 128, 128, 0, s>>>(n, j0, b, A);
      SG_CHECK_LAUNCH();
      // A22 -= L21 L21^T  (full square; only the lower part is used later)
      const double* L21 = A + int64_t(j0 + b) * n + j0;
      double* A22 = A + int64_t(j0 + b) * n + j0 + b;
      gemm(rows, rows, b, -1.0, L21, n, 1, L21, 1, n, 1.0, A22, n, 1, s);
    }
  }
  int h_info = 0;
  info.download(&h_info, 1, s);
  SG_CUDA(cudaStreamSynchronize(s));
  if (h_info) return false;
  // zero the strict upper triangle left over from the square trailing updates
  // (trsm / potrf wrote exact lower blocks; everything above the diagonal is junk)
  DBuf<double> Y(static_cast<size_t>(n) * n);
  identity_kernel<<<grid_blocks(int64_t(n) * n, 256), 256, 0, s>>>(n, Y.p);
  SG_CHECK_LAUNCH();
  // L Y = I, block rows top-down: Y_i = L_ii^-1 (I_i - L_i,<i Y_<i)
  for (int i0 = 0; i0 < n; i0 += kNB) {
    const int b = std::min(kNB, n - i0);
    const int ncols = i0 + b;  // Y is lower triangular
    if (i0 > 0) gemm(b, ncols, i0, -1.0, A + int64_t(i0) * n, n, 1, Y.p, n, 1, 1.0, Y.p + int64_t(i0) * n, n, 1, s);
    trsm_cols_kernel<<<(ncols + 127) / 128, 128, 0, s>>>(n, i0, b, ncols, A, Y.p);
    SG_CHECK_LAUNCH();
  }
  // A^-1 = Y^T Y
  gemm(n, n, n, 1.0, Y.p, 1, n, Y.p, n, 1, 0.0, Ainv, n, 1, s);
  SG_CUDA(cudaStreamSynchronize(s));
  return true;
}

}  // namespace sg
