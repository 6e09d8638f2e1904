// Device fixture generators: the reference's seeded
// density fields (states.py:58-111) drawn straight into HBM from the
// counter-based splitmix64 stream (prng.py:20-52).
//
// Draw n (n = 1, 2, ...) of a stream with seed s is mix(s + n * golden)
// (prng.py:20-41), so element e of an n-element field reads draw e + 1 and
// the second stream block of mixed_near_void reads draw n + e + 1: every
// element is independent and one thread makes one element.  uniform01 is
// (u64 >> 11) * 2^-53 (exact in double, prng.py:43-45); uniform is
// lo + (hi - lo) * u with numpy's two roundings (explicit _rn intrinsics, no
// FMA contraction).  The result is bit-identical to the host generators.
#include "sg_common.cuh"

namespace sg {
namespace {

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kMixA = 0xBF58476D1CE4E5B9ull;
constexpr unsigned long long kMixB = 0x94D049BB133111EBull;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(unsigned long long seed, unsigned long long ctr) {
  // (u64 >> 11) < 2^53 converts exactly; the scaling by 2^-53 is exact
  return __dmul_rn(__ull2double_rn(mix64(seed + kGolden * ctr) >> 11), 0x1.0p-53);
}

// kind: 0 uniform, 1 binary, 2 checkerboard, 3 layered, 4 random_floor,
// 5 mixed_near_void (states.py STATE_KINDS order)
__global__ void make_state_kernel(int kind, int nx, int ny, int64_t n, double vf, double floor_,
                                  unsigned long long seed, double* __restrict__ rho) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const unsigned long long ctr = static_cast<unsigned long long>(e) + 1ull;
  double v;
  switch (kind) {
    case 0: v = vf; break;
    case 1: v = u01(seed, ctr) < vf ? 1.0 : floor_; break;
    case 2: {
      const int64_t i = e % nx, j = (e / nx) % ny, k = e / (int64_t(nx) * ny);
      v = ((i + j + k) % 2 == 0) ? 1.0 : floor_;
      break;
    }
    case 3: {
      const int64_t j = (e / nx) % ny;
      v = (2 * j < ny) ? 1.0 : floor_;
      break;
    }
    case 4: v = __dadd_rn(floor_, __dmul_rn(__dsub_rn(1.0, floor_), u01(seed, ctr))); break;
    default: {
      const bool solid = u01(seed, ctr) < vf;
      const bool demote = u01(seed, static_cast<unsigned long long>(n) + ctr) < 0.1;
      v = (solid && !demote) ? 1.0 : floor_;
      break;
    }
  }
  rho[e] = v;
}

}  // namespace

void make_state_device(int kind, int nx, int ny, int nz, double vf, double floor_,
                       unsigned long long seed, double* rho, cudaStream_t s) {
  const int64_t n = int64_t(nx) * ny * nz;
  if (n == 0) return;
  make_state_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(kind, nx, ny, n, vf, floor_, seed, rho);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
