// On-device Galerkin coarse operators, bit-identical to the reference.
//
// Level 1 (transfer.py:129-174): per coarse element, sum of E_c * T_c over
// its 8 children (FMA-free, child order), then the Dirichlet corrections
// E_e * (masked - T) of boundary children; then the COO -> CSR pipeline of
// scipy (stable per-row placement, std::sort by column, sequential
// duplicate sums, exact-zero elimination) per row, with std::sort replayed
// exactly on device (sg_introsort.cuh).
//
// Levels >= 2 (transfer.py:177-181): canonical_csr(P^T (K P)) with scipy's
// csr_matmat summation orders: KP[j,k] = sum over sorted columns m of row j
// of K[j,m] P[m,k]; C[i,k] = sum over ascending j of KP[j,k] P[j,i].  P's
// weights are dyadic so every product is exact; sums are FMA-free.
#include <algorithm>
#include <set>
#include "sg_introsort.cuh"
#include "sg_kernels.cuh"

namespace sg {

// ------------------------------------------------------------ level 1
__global__ void boundary_code_kernel(GridDesc g, const uint8_t* __restrict__ nmask,
                                     uint32_t* __restrict__ codes) {
  const int64_t ne = g.nelem();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int ei = int(e % g.nx), ej = int((e / g.nx) % g.ny), ek = int(e / (int64_t(g.nx) * g.ny));
  const int NX = g.nx + 1, NY = g.ny + 1;
  uint32_t m24 = 0;
  for (int b = 0; b < 8; ++b) {
    const int ni = ei + (b & 1);
    const int64_t node = ni + int64_t(NX) * ((ej + ((b >> 1) & 1)) + int64_t(NY) * (ek + (b >> 2)));
    for (int a = 0; a < 3; ++a)
      if (node_fixed_axis(g, nmask, node, ni, a)) m24 |= 1u << (3 * b + a);
  }
  const uint32_t c = uint32_t((ei & 1) + 2 * (ej & 1) + 4 * (ek & 1));
  codes[e] = m24 ? ((c << 24) | m24) : 0u;
}

void boundary_codes(const FineOp& op, std::vector<uint32_t>& out, cudaStream_t s) {
  const int64_t ne = op.grid.d.nelem();
  DBuf<uint32_t> codes{size_t(ne)};
  boundary_code_kernel<<<grid_blocks(ne, 256), 256, 0, s>>>(op.grid.d, op.grid.nmask.p, codes.p);
  SG_CHECK_LAUNCH();
  std::vector<uint32_t> h(static_cast<size_t>(size_t(ne)));
  codes.download(h.data(), h.size(), s);
  SG_CUDA(cudaStreamSynchronize(s));
  std::set<uint32_t> uniq;
  for (uint32_t c : h)
    if (c) uniq.insert(c);
  out.assign(uniq.begin(), uniq.end());
}

__global__ void boundary_index_kernel(GridDesc g, const uint8_t* __restrict__ nmask,
                                      const uint32_t* __restrict__ table, int ntab,
                                      int16_t* __restrict__ bidx) {
  const int64_t ne = g.nelem();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int ei = int(e % g.nx), ej = int((e / g.nx) % g.ny), ek = int(e / (int64_t(g.nx) * g.ny));
  const int NX = g.nx + 1, NY = g.ny + 1;
  uint32_t m24 = 0;
  for (int b = 0; b < 8; ++b) {
    const int ni = ei + (b & 1);
    const int64_t node = ni + int64_t(NX) * ((ej + ((b >> 1) & 1)) + int64_t(NY) * (ek + (b >> 2)));
    for (int a = 0; a < 3; ++a)
      if (node_fixed_axis(g, nmask, node, ni, a)) m24 |= 1u << (3 * b + a);
  }
  int16_t r = -1;
  if (m24) {
    const uint32_t code = (uint32_t((ei & 1) + 2 * (ej & 1) + 4 * (ek & 1)) << 24) | m24;
    int lo = 0, hi = ntab - 1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (table[mid] == code) { r = int16_t(mid); break; }
      if (table[mid] < code) lo = mid + 1; else hi = mid - 1;
    }
  }
  bidx[e] = r;
}

// contrib[ce][a][b] (transfer.py:151-164)
__global__ void l1_contrib_kernel(GridDesc f, GridDesc c, const double* __restrict__ E,
                                  const int16_t* __restrict__ bidx, const double* __restrict__ tri,
                                  const double* __restrict__ diffs, double* __restrict__ contrib) {
  const int64_t total = c.nelem() * 576;
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= total) return;
  const int64_t ce = q / 576;
  const int ab = int(q % 576);
  const int ci = int(ce % c.nx), cj = int((ce / c.nx) % c.ny), ck = int(ce / (int64_t(c.nx) * c.ny));
  int64_t child[8];
#pragma unroll
  for (int ch = 0; ch < 8; ++ch)
    child[ch] = (2 * ci + (ch & 1)) + int64_t(f.nx) * ((2 * cj + ((ch >> 1) & 1)) + int64_t(f.ny) * (2 * ck + (ch >> 2)));
  double acc = 0.0;
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) acc = __dadd_rn(acc, __dmul_rn(E[child[ch]], tri[ch * 576 + ab]));
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const int bi = bidx[child[ch]];
    if (bi >= 0) acc = __dadd_rn(acc, __dmul_rn(E[child[ch]], diffs[int64_t(bi) * 576 + ab]));
  }
  contrib[q] = acc;
}

constexpr int kAsmThreads = 64;

// One thread per coarse node: COO stream of its rows -> std::sort replay ->
// sequential duplicate sums -> stencil slots (transfer.py:166-174, :33-39).
__global__ void __launch_bounds__(kAsmThreads) l1_assemble_kernel(GridDesc c, const uint8_t* __restrict__ cmask,
                                                                  const double* __restrict__ contrib,
                                                                  double* __restrict__ A) {
  extern __shared__ uint16_t sh_items[];
  const int64_t nn = c.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  uint16_t* items = sh_items + threadIdx.x * 192;
  const int NX = c.nx + 1, NY = c.ny + 1;
  const int i = int(node % NX), j = int((node / NX) % NY), k = int(node / (int64_t(NX) * NY));
  int n = 0;
  int64_t elem[8];
  int corner[8];
  for (int es = 0; es < 8; ++es) {
    const int di = (es & 1) - 1, dj = ((es >> 1) & 1) - 1, dk = (es >> 2) - 1;
    const int ei = i + di, ej = j + dj, ek = k + dk;
    elem[es] = -1;
    if (ei < 0 || ei >= c.nx || ej < 0 || ej >= c.ny || ek < 0 || ek >= c.nz) continue;
    elem[es] = ei + int64_t(c.nx) * (ej + int64_t(c.ny) * ek);
    corner[es] = -di + 2 * (-dj) + 4 * (-dk);
    for (int b = 0; b < 24; ++b) {
      const int cb = b / 3, ax = b % 3;
      const int ni = ei + (cb & 1), nj = ej + ((cb >> 1) & 1), nk = ek + (cb >> 2);
      const int64_t nb = ni + int64_t(NX) * (nj + int64_t(NY) * nk);
      if (node_fixed_axis(c, cmask, nb, ni, ax)) continue;
      const int slot = (nk - k + 1) * 9 + (nj - j + 1) * 3 + (ni - i + 1);
      items[n++] = uint16_t(((slot * 3 + ax) << 8) | (es * 24 + b));
    }
  }
  isort::sort(items, n);
  for (int ra = 0; ra < 3; ++ra) {
    if (node_fixed_axis(c, cmask, node, i, ra)) continue;
    int q = 0;
    while (q < n) {
      const int key = items[q] >> 8;
      double x = 0.0;
      bool first = true;
      while (q < n && (items[q] >> 8) == key) {
        const int id = items[q] & 0xFF;
        const int es = id / 24, b = id % 24;
        const double v = contrib[elem[es] * 576 + (3 * corner[es] + ra) * 24 + b];
        x = first ? v : __dadd_rn(x, v);
        first = false;
        ++q;
      }
      const int slot = key / 3, cax = key % 3;
      A[(int64_t(slot) * 9 + ra * 3 + cax) * nn + node] = x;
    }
  }
}

void galerkin_level1(const FineOp& op, const Grid& coarse, const L1Tables& t, double* A,
                     cudaStream_t s) {
  const GridDesc& f = op.grid.d;
  const GridDesc& c = coarse.d;
  const int64_t nf = f.nelem();
  const int nb = int(t.codes.size());
  DBuf<int16_t> bidx{size_t(nf)};
  DBuf<uint32_t> table{size_t(std::max(nb, 1))};
  DBuf<double> tri(8 * 576), diffs(size_t(std::max(nb, 1)) * 576);
  tri.upload(t.tri, 8 * 576, s);
  if (nb) {
    table.upload(t.codes.data(), size_t(nb), s);
    diffs.upload(t.diffs.data(), size_t(nb) * 576, s);
  }
  boundary_index_kernel<<<grid_blocks(nf, 256), 256, 0, s>>>(f, op.grid.nmask.p, table.p, nb, bidx.p);
  SG_CHECK_LAUNCH();
  const int64_t nce = c.nelem();
  DBuf<double> contrib(size_t(nce) * 576);
  l1_contrib_kernel<<<grid_blocks(nce * 576, 256), 256, 0, s>>>(f, c, op.E64.p, bidx.p, tri.p,
                                                                diffs.p, contrib.p);
  SG_CHECK_LAUNCH();
  const int64_t nn = c.nnodes();
  SG_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * 243 * nn, s));
  const size_t smem = size_t(kAsmThreads) * 192 * sizeof(uint16_t);
  l1_assemble_kernel<<<grid_blocks(nn, kAsmThreads), kAsmThreads, smem, s>>>(c, coarse.nmask.p,
                                                                            contrib.p, A);
  SG_CHECK_LAUNCH();
  SG_CUDA(cudaStreamSynchronize(s));  // temporaries die here
}

// ------------------------------------------------------- levels >= 2
__device__ __forceinline__ double w1d(int m, int k2) {
  const int d = m - k2;
  return d == 0 ? 1.0 : ((d == 1 || d == -1) ? 0.5 : 0.0);
}

// KP[((t*9 + ra*3 + cb) * nnf + j)], t = coarse offset slot relative to floor(j/2)-1.
__global__ void spgemm_kp_kernel(GridDesc f, GridDesc c, const uint8_t* __restrict__ cmask,
                                 const double* __restrict__ Af, double* __restrict__ KP) {
  const int64_t nnf = f.nnodes();
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nnf * 243) return;
  const int64_t j = q % nnf;
  const int r = int(q / nnf);
  const int t = r / 9, ra = (r / 3) % 3, cb = r % 3;
  const int FX = f.nx + 1, FY = f.ny + 1, CX = c.nx + 1, CY = c.ny + 1;
  const int jx = int(j % FX), jy = int((j / FX) % FY), jz = int(j / (int64_t(FX) * FY));
  const int kx = jx / 2 - 1 + t % 3, ky = jy / 2 - 1 + (t / 3) % 3, kz = jz / 2 - 1 + t / 9;
  double s = 0.0;
  if (kx >= 0 && kx <= c.nx && ky >= 0 && ky <= c.ny && kz >= 0 && kz <= c.nz) {
    const int64_t kn = kx + int64_t(CX) * (ky + int64_t(CY) * kz);
    if (!node_fixed_axis(c, cmask, kn, kx, cb)) {
      for (int slot = 0; slot < 27; ++slot) {
        const int mx = jx + slot % 3 - 1, my = jy + (slot / 3) % 3 - 1, mz = jz + slot / 9 - 1;
        if (mx < 0 || mx > f.nx || my < 0 || my > f.ny || mz < 0 || mz > f.nz) continue;
        const double w = w1d(mx, 2 * kx) * w1d(my, 2 * ky) * w1d(mz, 2 * kz);
        if (w == 0.0) continue;
        const double a = Af[(int64_t(slot) * 9 + ra * 3 + cb) * nnf + j];
        s = __dadd_rn(s, __dmul_rn(a, w));
      }
    }
  }
  KP[q] = s;
}

__global__ void spgemm_ptkp_kernel(GridDesc f, GridDesc c, const uint8_t* __restrict__ fmask,
                                   const uint8_t* __restrict__ cmask, const double* __restrict__ KP,
                                   double* __restrict__ Ac) {
  const int64_t nnc = c.nnodes(), nnf = f.nnodes();
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nnc * 243) return;
  const int64_t i = q % nnc;
  const int r = int(q / nnc);
  const int s2 = r / 9, ra = (r / 3) % 3, cb = r % 3;
  const int FX = f.nx + 1, FY = f.ny + 1, CX = c.nx + 1, CY = c.ny + 1;
  const int ix = int(i % CX), iy = int((i / CX) % CY), iz = int(i / (int64_t(CX) * CY));
  const int kx = ix + s2 % 3 - 1, ky = iy + (s2 / 3) % 3 - 1, kz = iz + s2 / 9 - 1;
  double s = 0.0;
  const bool ok = kx >= 0 && kx <= c.nx && ky >= 0 && ky <= c.ny && kz >= 0 && kz <= c.nz &&
                  !node_fixed_axis(c, cmask, i, ix, ra) &&
                  !node_fixed_axis(c, cmask, kx + int64_t(CX) * (ky + int64_t(CY) * kz), kx, cb);
  if (ok) {
    for (int dz = -1; dz <= 1; ++dz) {
      const int jz = 2 * iz + dz;
      if (jz < 0 || jz > f.nz) continue;
      const int tz = kz - (jz / 2 - 1);
      if (tz < 0 || tz > 2) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int jy = 2 * iy + dy;
        if (jy < 0 || jy > f.ny) continue;
        const int ty = ky - (jy / 2 - 1);
        if (ty < 0 || ty > 2) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int jx = 2 * ix + dx;
          if (jx < 0 || jx > f.nx) continue;
          const int tx = kx - (jx / 2 - 1);
          if (tx < 0 || tx > 2) continue;
          const int64_t j = jx + int64_t(FX) * (jy + int64_t(FY) * jz);
          if (node_fixed_axis(f, fmask, j, jx, ra)) continue;
          const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
          const int t = tz * 9 + ty * 3 + tx;
          const double v = KP[(int64_t(t) * 9 + ra * 3 + cb) * nnf + j];
          s = __dadd_rn(s, __dmul_rn(v, w));
        }
      }
    }
  }
  Ac[q] = s;
}

void galerkin_next(const Grid& fine, const Grid& coarse, const double* Af, double* Ac,
                   cudaStream_t s) {
  const int64_t nnf = fine.d.nnodes(), nnc = coarse.d.nnodes();
  DBuf<double> KP(size_t(nnf) * 243);
  spgemm_kp_kernel<<<grid_blocks(nnf * 243, 256), 256, 0, s>>>(fine.d, coarse.d, coarse.nmask.p,
                                                                Af, KP.p);
  SG_CHECK_LAUNCH();
  spgemm_ptkp_kernel<<<grid_blocks(nnc * 243, 256), 256, 0, s>>>(fine.d, coarse.d, fine.nmask.p,
                                                                 coarse.nmask.p, KP.p, Ac);
  SG_CHECK_LAUNCH();
  SG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sg
