// Common device/host helpers for the sm_100a PCG/GMG solver library.
//
// Data layout (all levels): a level vector lives in NODE layout, one
// contiguous array of 3 * n_nodes values (node = i + (nx+1)*(j + (ny+1)*k),
// dof = 3*node + axis, the reference's own DOF contract, grid.py:3-8).
// Fixed (Dirichlet) DOFs are held at exactly zero, so the free-DOF vectors of
// the reference API are a gather of this array (free2dof).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace sg {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SG_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      (void)cudaGetLastError(); /* a non-sticky API error must not resurface */    \
      throw ::sg::Error(std::string("CUDA error ") + cudaGetErrorString(_e) +     \
                        " at " __FILE__ ":" + std::to_string(__LINE__));           \
    }                                                                              \
  } while (0)

// Every kernel launch of the library is followed by SG_CHECK_LAUNCH(), which
// also counts it (sg_launch_count(): evidence of native launches per step).
extern unsigned long long g_sg_launches;
#define SG_CHECK_LAUNCH()                                 \
  do {                                                    \
    __atomic_add_fetch(&::sg::g_sg_launches, 1ull, __ATOMIC_RELAXED); \
    SG_CUDA(cudaGetLastError());                          \
  } while (0)

#define SG_REQUIRE(cond, msg)                                                      \
  do {                                                                             \
    if (!(cond)) throw ::sg::Error(msg);                                           \
  } while (0)

// SM count of the current device (148 on a full B200; fewer under MIG / MPS
// SM limits), queried once per device.
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    SG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = n > 0 ? n : 1;
  }
  return cache[dev];
}

// Owning device buffer (cudaMalloc'd, freed on destruction).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) SG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void zero(cudaStream_t s) {
    if (n) SG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* host, size_t count, cudaStream_t s) {
    SG_REQUIRE(count <= n, "upload overflow");
    if (count) SG_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* host, size_t count, cudaStream_t s) const {
    SG_REQUIRE(count <= n, "download overflow");
    if (count) SG_CUDA(cudaMemcpyAsync(host, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
};

// Structured grid of one hierarchy level: element counts, a per-node 3-bit
// Dirichlet mask and the free<->dof maps used at the API boundary.
struct GridDesc {
  int nx = 0, ny = 0, nz = 0;
  bool xface = false;  // mask == "every DOF of the x=0 face fixed, nothing else"
  __host__ __device__ int64_t nnodes() const {
    return int64_t(nx + 1) * (ny + 1) * (nz + 1);
  }
  __host__ __device__ int64_t nelem() const { return int64_t(nx) * ny * nz; }
};

struct Grid {
  GridDesc d;
  int64_t n_free = 0;
  DBuf<uint8_t> nmask;     // per node: bit a set => axis a fixed
  DBuf<int32_t> free2dof;  // n_free
  DBuf<int32_t> dof2free;  // 3*nnodes, -1 for fixed
  std::vector<uint8_t> h_nmask;
};

__device__ __forceinline__ bool node_fixed_axis(const GridDesc& g, const uint8_t* nmask,
                                                int64_t node, int i, int axis) {
  if (g.xface) return i == 0;
  return (nmask[node] >> axis) & 1;
}

inline int grid_blocks(int64_t n, int threads, int64_t cap = 1 << 30) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return int(b);
}

// bf16 round-to-nearest-even on the FP32 bit pattern (precision.py:25-48),
// NaN passes through unchanged.
__host__ __device__ __forceinline__ float bf16_round(float x) {
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) return x;
  uint32_t r = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  return __uint_as_float(r);
#else
  uint32_t b;
  memcpy(&b, &x, 4);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) return x;
  uint32_t r = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  float o;
  memcpy(&o, &r, 4);
  return o;
#endif
}

}  // namespace sg
