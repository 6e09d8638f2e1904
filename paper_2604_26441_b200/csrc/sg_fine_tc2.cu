// Level-0 apply under the BF16EMU tag on the 5th-generation tensor cores,
// pipelined (fine_operator.py:71-72: local = round_bf16(u_e) @ round_bf16(Ke32),
// FP32 accumulation, the element modulus applied after the contraction).
//
// The element-major GEMM (M = elements, K = 24 corner DOFs, N = 24 outputs) is
// fed WITHOUT per-element operand staging: a node plane is written to shared
// memory once as 16-byte "records", record (row j, column i) = BF16 of
// [u(i-1, j), u(i, j)] (6 values + 2 zeros = one 8-wide K chunk of a UMMA core
// matrix).  The A operand of a 128-element tile of one layer is then a plain
// descriptor over consecutive records: K chunk 0 = records of node row j
// (corners y = 0), K chunk 1 = records of row j + 1 at LBO = one record row
// (corners y = 1), 8-record core-matrix groups at SBO = 128 B.  Two
// tcgen05.mma (K = 16 each, kind::f16, BF16 x BF16 -> FP32 in TMEM) per tile
// cover the z = 0 and z = 1 corner planes; B = the matching rows of
// round_bf16(Ke), fixed for the launch.  Elements are flattened row-major over
// the CTA's element rows with one phantom column per row (modulus 0), so rows
// chain without gaps and x-neighbours are adjacent tile rows.
//
// Pipeline per layer (512 threads, three block barriers):
//   A  records of node plane k+1 from its FP32 staging buffer (BF16 rounding
//      once per node, not once per element corner);
//   B  barrier; one thread issues the layer's MMAs into TMEM buffer k&1 and
//      commits them to that buffer's mbarrier;
//   D  epilogue of layer k-1 while the MMAs of layer k run: tcgen05.ld of the
//      accumulators, modulus scaling, x-neighbour corners by warp shuffle, the
//      "up" partials published in shared memory, barrier, each owned node
//      summed in a fixed order ((own + right) + (up + up-right), then + the
//      layer below) and stored;
//   C  node plane k+3 and layer k+3's moduli staged by cp.async (three
//      buffers: two planes in flight behind the one being recorded), barrier.
// BF16 x BF16 products are exact in FP32, so only the FP32 summation order
// differs from the reference's sgemm (tolerance parity).
#include "sg_kernels.cuh"

namespace sg {

namespace {

constexpr int kT2Threads = 512;               // record / epilogue warps
constexpr int kT2Block = kT2Threads + 32;      // + one MMA-issuing warp
constexpr int kT2MaxTiles = 8;  // TMEM: 2 buffers x 8 tiles x 32 columns = 512

__device__ __forceinline__ uint32_t sm_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, no swizzle: start | LBO (K-chunk stride) | SBO (8-row group stride) | version 1
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// kind::f16: D = F32, A = B = BF16, both K-major, N = 32, M = 128
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t bf16u(float x) {
  return __float_as_uint(bf16_round(x)) >> 16;
}
// two values rounded to BF16 (nearest, ties to even: the bits of bf16_round for
// every non-NaN input) in one cvt.rn.bf16x2.f32; lo = a
__device__ __forceinline__ uint32_t bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

}  // namespace

__global__ void __launch_bounds__(kT2Block, 1)
fine_bf16_tc2_kernel(GridDesc g, const uint8_t* __restrict__ nmask, const float* __restrict__ u,
                     float* __restrict__ y, const float* __restrict__ E, KeParam<float> ke16, int R,
                     int T, int kchunk) {
  extern __shared__ __align__(1024) uint8_t sm2[];
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int nE = R * NX;                 // element slots (row-major, one phantom column)
  const int nRec = (R + 1) * NX;         // records of one node plane
  const int RS = T * 128 + NX + 8;       // record slot length (zero tail for the last tile)
  const int PS = T * 128 + 32;           // published-partials stride
  const int F3 = 3 * NX;                 // floats per node row
  const int nflt = (R + 1) * F3;         // floats of one staging plane
  const int SS = (nflt + 3) & ~3;
  uint8_t* sB = sm2;                                      // 2 x 1 KB (z = 0, 1)
  uint4* rec = reinterpret_cast<uint4*>(sm2 + 2048);      // [3][RS] records
  float* stg = reinterpret_cast<float*>(rec + 3 * RS);    // [3][SS] FP32 node planes (cp.async)
  float* est = stg + 3 * SS;                              // [4][T*128] element moduli (cp.async)
  float* pub = est + 4 * T * 128;                         // [6][PS] "up" partials
  float* edge = pub + 6 * PS;                             // [T*4 + 1][12] lane-0 corners of 32-blocks
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int y0 = int(blockIdx.x) * (R - 1);  // first owned node row; node row r <-> y0 - 1 + r
  const int k0 = int(blockIdx.y) * kchunk;
  const int k1 = min(k0 + kchunk, g.nz + 1);  // output node planes [k0, k1)
  const int64_t plane = int64_t(3) * NX * NY;
  const int64_t estride = int64_t(g.nx) * g.ny;

  // ---- setup: records / staging zeroed (tails and out-of-grid rows stay 0),
  // B tiles, mbarriers, TMEM
  for (int q = tid; q < 3 * RS; q += kT2Block) rec[q] = make_uint4(0u, 0u, 0u, 0u);
  for (int q = tid; q < 3 * SS + 4 * T * 128 + 6 * PS + (T * 4 + 1) * 12; q += kT2Block) stg[q] = 0.0f;
  for (int q = tid; q < 2 * 32 * 16; q += kT2Block) {
    const int cz = q >> 9, n = (q >> 4) & 31, k = q & 15;
    const int cy = k >> 3, kk = k & 7, cx = kk / 3, c = kk % 3;
    float v = 0.0f;
    if (n < 24 && kk < 6) v = ke16.k[(3 * (cx + 2 * cy + 4 * cz) + c) * 24 + n];  // B[n][k] = Ke[dof][n]
    *reinterpret_cast<uint16_t*>(sB + cz * 1024 + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 +
                                 (k & 7) * 2) = uint16_t(bf16u(v));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sm_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  // ---- this thread's element slots: tiles m = (warp >> 2) + 4 a, row 32 (warp & 3) + lane
  const int q4 = warp & 3, m0 = warp >> 2;
  constexpr int kA = (kT2MaxTiles + kT2Threads / 128 - 1) / (kT2Threads / 128);  // tiles per thread
  int tt[kA], eo[kA];       // slot, element offset in its layer (-1: no element)
  bool ownn[kA];
  int64_t onode[kA];
#pragma unroll
  for (int a = 0; a < kA; ++a) {
    const int t = (m0 + 4 * a) * 128 + q4 * 32 + lane;
    const int r = t / NX, i = t - r * NX;
    const int ex = i - 1, ej = y0 - 1 + r, nj = y0 + r;
    tt[a] = t;
    eo[a] = (t < nE && ex >= 0 && ex < g.nx && ej >= 0 && ej < g.ny) ? ex + g.nx * ej : -1;
    ownn[a] = t < nE && r <= R - 2 && nj <= g.ny;
    onode[a] = int64_t(i) + int64_t(NX) * min(nj, g.ny);
  }

  // ---- async staging of node plane kp (rows y0-1 .. y0+R-1, contiguous) into
  // buffer kp mod 3 and of layer kp's moduli into buffer kp mod 4 (read by the
  // epilogue of layer kp one iteration after stage(kp + 3)); out-of-grid
  // entries stay 0
  auto stage = [&](int kp) {
    const int sb = ((kp % 3) + 3) % 3;
    if (kp >= 0 && kp <= g.nz) {
      const int jlo = max(y0 - 1, 0), jhi = min(y0 - 1 + R, g.ny);  // valid node rows
      const int r0 = jlo - (y0 - 1);
      const float* src = u + int64_t(kp) * plane + int64_t(F3) * jlo;
      float* dst = stg + sb * SS + r0 * F3;
      const int n = (jhi - jlo + 1) * F3;
      for (int q = tid; q < n; q += kT2Threads)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sm_u32(dst + q)), "l"(src + q) : "memory");
    }
    if (kp >= 0 && kp < g.nz) {
#pragma unroll
      for (int a = 0; a < kA; ++a)
        if (eo[a] >= 0)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sm_u32(est + (kp & 3) * T * 128 + tt[a])),
                       "l"(E + eo[a] + int64_t(kp) * estride) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // this thread's records q = tid + 512 k: smem offset of node (i, r) in the
  // staging plane (fixed for the launch: no divisions in the layer loop)
  constexpr int kRecPer = 4;
  int roff[kRecPer];
#pragma unroll
  for (int k = 0; k < kRecPer; ++k) {
    const int q = tid + k * kT2Threads;
    const int r = q / NX, i = q - r * NX;
    roff[k] = q < nRec ? (r * F3 + 3 * i) | (i > 0 ? 0 : int(0x80000000u)) : -1;
  }
  auto build_records = [&](int kp) {  // staging plane kp -> record slot kp mod 3
    const int sb = ((kp % 3) + 3) % 3;
    uint4* rs = rec + sb * RS;
    const float* st = stg + sb * SS;
    const bool in = kp >= 0 && kp <= g.nz;
#pragma unroll
    for (int k = 0; k < kRecPer; ++k) {
      if (roff[k] == -1) break;
      const int q = tid + k * kT2Threads;
      const int i = roff[k] < 0 ? 0 : 1;  // 0: first column (no left node)
      const float* row = st + (roff[k] & 0x7FFFFFFF);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f;
      if (in) {
        if (i > 0) {
          a0 = row[-3];
          a1 = row[-2];
          a2 = row[-1];
        }
        b0 = row[0];
        b1 = row[1];
        b2 = row[2];
      }
      rs[q] = make_uint4(bf16x2(a0, a1), bf16x2(a2, b0), bf16x2(b1, b2), 0u);
    }
  };

  float carry[kA][3];
#pragma unroll
  for (int a = 0; a < kA; ++a) carry[a][0] = carry[a][1] = carry[a][2] = 0.0f;
  uint32_t phase[2] = {0u, 0u};

  auto epilogue = [&](int ek) {  // layer ek: accumulators in TMEM buffer ek & 1
    const int b = ek & 1;
    const int sb = ek & 3;  // moduli buffer
    const bool kin = ek >= 0 && ek < g.nz;
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(sm_u32(&mbar[b])), "r"(phase[b]));
      }
      phase[b] ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    float own[kA][6], right[kA][6];
#pragma unroll
    for (int a = 0; a < kA; ++a) {
      const int m = m0 + 4 * a;
      if (m >= T) break;  // warp-uniform
      const int t = tt[a];
      uint32_t d[24];
      const uint32_t ta = tmem + (uint32_t(q4 * 32) << 16) + uint32_t(b * T * 32 + m * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
            "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
            "=r"(d[14]), "=r"(d[15])
          : "r"(ta));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
                     "=r"(d[22]), "=r"(d[23])
                   : "r"(ta + 16u));
      const float e = (kin && eo[a] >= 0) ? est[sb * T * 128 + t] : 0.0f;
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float w[24];
#pragma unroll
      for (int n = 0; n < 24; ++n) w[n] = __uint_as_float(d[n]) * e;
      // corner (cx, cy, cz) -> w[3 (cx + 2 cy + 4 cz) + c]; "up" = (1,0)(t) + (0,0)(t+1)
#pragma unroll
      for (int cz = 0; cz < 2; ++cz)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float r01 = w[3 * (2 + 4 * cz) + c], r10 = w[3 * (1 + 4 * cz) + c],
                      r00 = w[3 * (0 + 4 * cz) + c];
          own[a][3 * cz + c] = w[3 * (3 + 4 * cz) + c];
          right[a][3 * cz + c] = __shfl_down_sync(0xffffffffu, r01, 1);
          const float n00 = __shfl_down_sync(0xffffffffu, r00, 1);
          pub[(3 * cz + c) * PS + t] = lane < 31 ? r10 + n00 : r10;
          if (lane == 0) {
            edge[(t >> 5) * 12 + 3 * cz + c] = r01;
            edge[(t >> 5) * 12 + 6 + 3 * cz + c] = r00;
          }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("bar.sync 2, %0;" ::"n"(kT2Threads) : "memory");  // compute warps
    // owned nodes: element (i, r) owns node (i, y0 + r):
    //   ((own (1,1) + right (0,1)) + (up (1,0) + up-right (0,0))), then carry + z = 0 part
#pragma unroll
    for (int a = 0; a < kA; ++a) {
      const int m = m0 + 4 * a;
      if (m >= T || !ownn[a]) continue;
      const int t = tt[a], tu = t + NX;
      const bool last_u = (tu & 31) == 31;
      float v[2][3];
#pragma unroll
      for (int cz = 0; cz < 2; ++cz)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float rr = lane < 31 ? right[a][3 * cz + c] : edge[((t + 1) >> 5) * 12 + 3 * cz + c];
          const float lo = own[a][3 * cz + c] + rr;
          float hi = pub[(3 * cz + c) * PS + tu];
          if (last_u) hi = hi + edge[((tu + 1) >> 5) * 12 + 6 + 3 * cz + c];
          v[cz][c] = lo + hi;
        }
      if (ek >= k0) {
        const int64_t node = onode[a] + int64_t(ek) * NX * NY;
        const unsigned fm = g.xface ? ((t % NX) == 0 ? 7u : 0u) : unsigned(nmask[node]);
        float* yp = y + 3 * node;
#pragma unroll
        for (int c = 0; c < 3; ++c) yp[c] = ((fm >> c) & 1u) ? 0.0f : carry[a][c] + v[0][c];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) carry[a][c] = v[1][c];
    }
  };

  if (warp == kT2Threads / 32) {
    // ---- MMA warp: layer ek's MMAs once the records of plane ek+1 exist and
    // the TMEM buffer ek&1 was drained (epilogue of ek-2 precedes the arrive)
    const uint64_t bd0 = umma_desc(sm_u32(sB), 128, 256), bd1 = umma_desc(sm_u32(sB + 1024), 128, 256);
    for (int ek = k0 - 1; ek < k1; ++ek) {
      asm volatile("bar.sync 1, %0;" ::"n"(kT2Block) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t b = uint32_t(ek & 1);
        const int s0 = ((ek % 3) + 3) % 3, s1 = (((ek + 1) % 3) + 3) % 3;
        const uint32_t ra = sm_u32(rec + s0 * RS), rb = sm_u32(rec + s1 * RS);
        const uint64_t a0 = umma_desc(ra, uint32_t(NX) * 16u, 128), a1 = umma_desc(rb, uint32_t(NX) * 16u, 128);
        for (int m = 0; m < T; ++m) {
          const uint32_t dt = tmem + b * uint32_t(T * 32) + uint32_t(m * 32);
          const uint64_t dm = uint64_t(m) * (2048u >> 4);  // start address field, + m tiles
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
              ::"r"(dt), "l"(a0 + dm), "l"(bd0), "r"(kIdesc2), "r"(0u));
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
              ::"r"(dt), "l"(a1 + dm), "l"(bd1), "r"(kIdesc2), "r"(1u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(sm_u32(&mbar[b])));
      }
      __syncwarp();
    }
  } else {
    // ---- record / epilogue warps.  Prologue: planes k0-1, k0 staged and
    // recorded, k0+1 in flight
    stage(k0 - 1);
    stage(k0);
    stage(k0 + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    asm volatile("bar.sync 3, %0;" ::"n"(kT2Threads) : "memory");
    build_records(k0 - 1);
    for (int ek = k0 - 1; ek < k1; ++ek) {
      // A: records of node plane ek+1 (staged, waited and barriered last layer)
      build_records(ek + 1);
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      // B: hand layer ek to the MMA warp (no wait)
      asm volatile("bar.arrive 1, %0;" ::"n"(kT2Block) : "memory");
      // D: epilogue of the previous layer while layer ek's MMAs run
      if (ek > k0 - 1) epilogue(ek - 1);
      // C: stage node plane ek+3 into the buffer of plane ek (recorded last
      // layer; in the first layer by the prologue, with no epilogue barrier
      // since -- wait for every thread's reads of it first)
      if (ek == k0 - 1) asm volatile("bar.sync 3, %0;" ::"n"(kT2Threads) : "memory");
      stage(ek + 3);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // plane ek+2 landed
      asm volatile("bar.sync 3, %0;" ::"n"(kT2Threads) : "memory");
    }
    epilogue(k1 - 1);
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Tiling: R element rows per CTA (R - 1 owned node rows) with R * NX <= 1024
// element slots (8 tiles of 128), z chunks minimising waves x (chunk + 1).
// false: the grid is too wide for this kernel (NX > 512 or the staging plane
// exceeds the per-thread budget) -- the caller runs the per-element kernel.
bool bf16_tc2_plan(const GridDesc& g, int nsm, int& R, int& T, int& ty, int& kchunk, int& nch,
                   size_t& smem) {
  const int NX = g.nx + 1, NY = g.ny + 1, planes = g.nz + 1;
  R = std::min(kT2MaxTiles * 128 / NX, NY + 1);
  if (R < 2) return false;
  T = (R * NX + 127) / 128;
  ty = (NY + R - 2) / (R - 1);
  long best = 1L << 60;
  nch = 1;
  for (int c = 1; c <= planes; ++c) {
    const int kc = (planes + c - 1) / c;
    const int n = (planes + kc - 1) / kc;
    const long waves = (long(ty) * n + nsm - 1) / nsm;
    const long cost = waves * (kc + 1);
    if (cost < best) { best = cost; nch = n; }
  }
  kchunk = (planes + nch - 1) / nch;
  nch = (planes + kchunk - 1) / kchunk;
  const int RS = T * 128 + NX + 8, PS = T * 128 + 32, SS = ((R + 1) * 3 * NX + 3) & ~3;
  smem = 2048 + size_t(3) * RS * 16 +
         sizeof(float) * (size_t(3) * SS + size_t(4) * T * 128 + size_t(6) * PS + size_t(T * 4 + 1) * 12);
  return smem <= 220 * 1024;
}

bool fine_apply_bf16_tc2(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  const GridDesc& g = op.grid.d;
  int R, T, ty, kchunk, nch;
  size_t smem;
  if (!bf16_tc2_plan(g, num_sms(), R, T, ty, kchunk, nch, smem)) return false;
  static size_t attr = 0;
  if (smem > attr) {
    SG_CUDA(cudaFuncSetAttribute(fine_bf16_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    attr = smem;
  }
  fine_bf16_tc2_kernel<<<dim3(ty, nch), kT2Block, smem, s>>>(g, op.grid.nmask.p, u, y, op.E32.p,
                                                               op.ke16, R, T, kchunk);
  SG_CHECK_LAUNCH();
  return true;
}

}  // namespace sg
