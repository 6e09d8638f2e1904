// Level-0 apply under the BF16EMU tag on the 5th-generation tensor cores
// (reference: fine_operator.py:71-72, local = round_bf16(u_e) @ round_bf16(Ke32),
// FP32 accumulation, modulus applied after the contraction).
//
// Same z-streaming decomposition as the Walsh FP32/FP64 kernel (16x16 element
// columns per CTA, one element per thread per layer, deterministic x/y/z
// corner combination), but the 24x24 contraction of the 256 elements of a
// layer is two tcgen05.mma.kind::f16 instructions (M=128 elements, N=32
// output DOFs (24 used), K=32 (24 used), BF16 x BF16 -> FP32 in TMEM):
//   * each thread writes its element's 24 BF16-rounded values into the UMMA
//     canonical K-major (no swizzle) core-matrix layout in shared memory;
//   * one elected thread issues the MMAs and commits them to an mbarrier;
//   * each warp reads its 32 TMEM lanes (tcgen05.ld 32x32b.x32): lane = element,
//     columns = the element's 24 local results; E is applied in FP32.
// BF16 x BF16 products are exact in FP32, so only the FP32 summation order
// differs from the reference's sgemm (tolerance parity).
#include "sg_kernels.cuh"

namespace sg {

namespace {

constexpr int kTX = 16, kTY = 16, kTThreads = kTX * kTY;
// UMMA canonical K-major / SWIZZLE_NONE layout: 8-row x 16-byte core matrices,
// k-chunks of 8 BF16 at +128 B (LBO), 8-row groups at +512 B (SBO).
constexpr int kRowBytes = 64;            // 32 BF16 per row (24 used)
constexpr int kTileBytes = 128 * kRowBytes;  // one M=128 operand tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t core_off(int row, int k) {
  return uint32_t((row >> 3) * 512 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  // start >> 4 | LBO (128 B) >> 4 << 16 | SBO (512 B) >> 4 << 32 | version 1 << 46 | SWIZZLE_NONE
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(512 >> 4) << 32) |
         (uint64_t(1) << 46);
}

// kind::f16 instruction descriptor: D=F32, A=B=BF16, K-major both, N=32, M=128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  return uint16_t(__float_as_uint(bf16_round(x)) >> 16);
}

}  // namespace

__global__ void __launch_bounds__(kTThreads, 1)
fine_apply_bf16_tc_kernel(GridDesc g, const uint8_t* __restrict__ nmask, const float* __restrict__ u,
                          float* __restrict__ y, const float* __restrict__ E, KeParam<float> ke16,
                          int kchunk) {
  __shared__ __align__(1024) uint8_t sA[2 * kTileBytes];   // two M=128 element tiles
  __shared__ __align__(1024) uint8_t sB[32 * kRowBytes];   // Ke (N=32 x K=32)
  __shared__ float ex[2][kTY][kTX][6];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int tx = tid & (kTX - 1), ty = tid / kTX;
  const int ei = int(blockIdx.x) * (kTX - 1) - 1 + tx;
  const int ej = int(blockIdx.y) * (kTY - 1) - 1 + ty;
  const int k0 = int(blockIdx.z) * kchunk;
  const int k1 = min(k0 + kchunk, g.nz + 1);
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int ni = ei + 1, nj = ej + 1;
  const bool own = tx < kTX - 1 && ty < kTY - 1 && ni <= g.nx && nj <= g.ny;
  const bool col_in = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny;
  const int ci0 = min(max(ei, 0), g.nx), ci1 = min(max(ei + 1, 0), g.nx);
  const int cj0 = min(max(ej, 0), g.ny), cj1 = min(max(ej + 1, 0), g.ny);
  const int off1 = 3 * (ci1 - ci0), off2 = 3 * NX * (cj1 - cj0);
  const int64_t plane = 3 * int64_t(NX) * NY;
  const float* ucol = u + 3 * (int64_t(ci0) + int64_t(NX) * cj0);
  const int64_t estride = int64_t(g.nx) * g.ny;
  const float* ecol = E + (col_in ? ei + int64_t(g.nx) * ej : 0);
  const bool xface_fixed = g.xface && ni == 0;
  float* yp = y + 3 * (int64_t(min(ni, g.nx)) + int64_t(NX) * min(nj, g.ny)) + int64_t(k0) * plane;
  const uint8_t* mp = nmask ? nmask + (int64_t(min(ni, g.nx)) + int64_t(NX) * min(nj, g.ny)) +
                                  int64_t(k0) * NX * NY : nullptr;

  // ---- one-time setup: B operand, mbarrier, TMEM (64 columns: two 32-col accumulators)
  for (int q = tid; q < 32 * 32; q += kTThreads) {
    const int n = q / 32, k = q % 32;
    const float v = (n < 24 && k < 24) ? ke16.k[k * 24 + n] : 0.0f;  // B[n][k] = Ke[k][n]
    *reinterpret_cast<uint16_t*>(sB + core_off(n, k)) = bf16_bits(v);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto load_plane = [&](int kp, float* dst) {
    const float* p = ucol + int64_t(min(max(kp, 0), g.nz)) * plane;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dst[c] = __ldg(p + c);
      dst[3 + c] = __ldg(p + off1 + c);
      dst[6 + c] = __ldg(p + off2 + c);
      dst[9 + c] = __ldg(p + off2 + off1 + c);
    }
  };
  float lo[12], hi[12];
  load_plane(k0 - 1, lo);
  float carry[3] = {0.f, 0.f, 0.f};
  int buf = 0;
  uint32_t phase = 0;
  const int region = tid >> 7, row = tid & 127;
  uint8_t* myrow = sA + region * kTileBytes;
  for (int ek = k0 - 1; ek < k1; ++ek) {
    load_plane(ek + 1, hi);
    const bool el_ok = col_in && ek >= 0 && ek < g.nz;
    const float s = el_ok ? __ldg(ecol + int64_t(min(max(ek, 0), g.nz - 1)) * estride) : 0.0f;
    // stage this element's 24 BF16-rounded inputs (corners 0..3 = lo, 4..7 = hi)
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      uint32_t w[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int k0i = kc * 8 + 2 * h, k1i = k0i + 1;
        auto val = [&](int k) -> float {
          if (k >= 24) return 0.0f;
          const int corner = k / 3, c = k % 3;
          return corner < 4 ? lo[3 * corner + c] : hi[3 * (corner - 4) + c];
        };
        w[h] = uint32_t(bf16_bits(val(k0i))) | (uint32_t(bf16_bits(val(k1i))) << 16);
      }
      *reinterpret_cast<uint4*>(myrow + core_off(row, kc * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ad = smem_desc(smem_u32(sA + r * kTileBytes) + ks * 256);
          const uint64_t bd = smem_desc(smem_u32(sB) + ks * 256);
          const uint32_t acc = ks > 0 ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
              ::"r"(tmem + uint32_t(r * 32)), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&mbar)));
    }
    // wait for the accumulators
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[32];
    const uint32_t taddr = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(region * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
          "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]),
          "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]),
          "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    float w[24];
#pragma unroll
    for (int q = 0; q < 24; ++q) w[q] = __uint_as_float(d[q]) * s;  // modulus after the contraction
    // x-combine (warp shuffle), y-combine (shared memory), z-combine (registers)
    float A[12];
#pragma unroll
    for (int jy = 0; jy < 2; ++jy)
#pragma unroll
      for (int kz = 0; kz < 2; ++kz)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int cr = 1 + 2 * jy + 4 * kz, cl = 2 * jy + 4 * kz;
          A[(jy * 2 + kz) * 3 + c] = w[3 * cr + c] + __shfl_down_sync(0xffffffffu, w[3 * cl + c], 1, 16);
        }
#pragma unroll
    for (int t = 0; t < 6; ++t) ex[buf][ty][tx][t] = A[t];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    const bool up = ty < kTY - 1;
    float B[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) B[t] = up ? A[6 + t] + ex[buf][ty + 1][tx][t] : A[6 + t];
    buf ^= 1;
    if (ek >= k0) {
      if (own) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const bool fixed = g.xface ? xface_fixed : ((mp[0] >> c) & 1);
          yp[c] = fixed ? 0.0f : carry[c] + B[c];
        }
      }
      yp += plane;
      if (!g.xface) mp += int64_t(NX) * NY;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) carry[c] = B[3 + c];
#pragma unroll
    for (int q = 0; q < 12; ++q) lo[q] = hi[q];
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

void fine_apply_bf16_tc(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  const GridDesc& g = op.grid.d;
  const int tx = (g.nx + 1 + kTX - 2) / (kTX - 1);
  const int ty = (g.ny + 1 + kTY - 2) / (kTY - 1);
  const int planes = g.nz + 1;
  int nchunk = std::max(1, std::min((2 * num_sms() + tx * ty - 1) / (tx * ty), (planes + 3) / 4));
  const int kchunk = (planes + nchunk - 1) / nchunk;
  nchunk = (planes + kchunk - 1) / kchunk;
  dim3 grid(tx, ty, nchunk);
  fine_apply_bf16_tc_kernel<<<grid, kTThreads, 0, s>>>(g, op.grid.nmask.p, u, y, op.E32.p, op.ke16, kchunk);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
