// Device-side slab transport ("overlap
// exchange on the fine matrix-free action"): the three data movements of the
// slab-partitioned solve -- ghost-plane exchange, rank-ordered sum of a few
// doubles, allgather of owned planes -- as stream-ordered kernels that store
// straight into the peer ranks' memory (CUDA IPC mappings over NVLink / the
// same device) and signal with release/acquire flags at system scope.  No
// host round trip, so the distributed V-cycle is CUDA-graph capturable.
//
// Every rank owns one "mailbox" allocation laid out identically on all ranks:
//   halo slots  [level][parity][src]  (ghost planes a source sends this rank)
//   sum slots   [parity][src][8]      (per-rank partials of an allreduce)
//   gather slot [parity][full level]  (owned planes of every rank, in place)
//   flags       halo[src], halo_ack[dst], sum[src], gather[src]  (u64 epochs)
// An exchange of epoch e: the sender waits until the receiver has released
// the slot it is about to reuse (halo_ack >= e - 2; parity double buffering),
// stores its planes into the receiver's slot, fences at system scope and
// raises halo[me] = e in the receiver's flags (one release store by the last
// block to finish); the receiver's pull kernel acquires the flags and copies
// the slot into its ghost planes, then acks.  Sums and gathers are all-to-all,
// so a rank cannot lap a slot another rank still reads (its epoch e + 2 push
// needs that rank's epoch e + 1 push, which follows its epoch e read).  The
// epochs live in device memory and advance inside the kernels: graph replays
// stay in step.  Sums are accumulated in rank order: identical bits on every
// rank, as TorchSlabComm.allreduce.
#include <cstdio>
#include <cstring>
#include "sg_hier.cuh"
#include "sg_peer.cuh"

namespace sg {

namespace {

enum { CH_HALO = PEER_CH_HALO, CH_SUM = PEER_CH_SUM, CH_GATHER = PEER_CH_GATHER };
constexpr int kMaxRanks = kPeerMaxRanks;
constexpr int kMaxXfer = 8;   // sends or receives of one rank on one level
constexpr int kSumMax = kPeerSumMax;

__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) { return peer_ld_acq(p); }
__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) { peer_st_rel(p, v); }
__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long v) { peer_wait_geq(p, v); }

struct Xfer {          // one contiguous plane range
  int n = 0;
  int peer[kMaxXfer];  // destination (push) / source (pull) rank
  long long src_off[kMaxXfer], dst_off[kMaxXfer], count[kMaxXfer];  // in elements
  long long total = 0;
};

struct PeerPtrs {
  char* base[kMaxRanks];
};

// last block of the grid (all earlier blocks' stores fenced) -> true
__device__ __forceinline__ bool last_block(unsigned* arrive) {
  __shared__ bool last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned n = atomicAdd(arrive, 1u);
    last = n == gridDim.x - 1;
    if (last) *arrive = 0u;
  }
  __syncthreads();
  return last;
}

template <class T>
__device__ __forceinline__ void copy_ranges(const Xfer& X, const T* src, T* const* dst_base,
                                            bool cg_src) {
  for (long long i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < X.total;
       i += int64_t(gridDim.x) * blockDim.x) {
    long long k = i;
    int j = 0;
    while (k >= X.count[j]) k -= X.count[j++];
    const T* sp = src + X.src_off[j] + k;
    const T v = cg_src ? __ldcg(sp) : *sp;
    dst_base[j][X.dst_off[j] + k] = v;
  }
}

// halo push: my owned planes -> the receivers' slots (slot offsets in dst_off)
template <class T>
__device__ __forceinline__ void halo_push(const Xfer& X, const T* __restrict__ vec, const PeerPtrs& P, int me,
                                 size_t slot_level_off, size_t slot_bytes, int world,
                                 size_t flags_off, unsigned long long* ep, unsigned* arrive) {
  const unsigned long long e = ep[CH_HALO] + 1;
  const int par = int(e & 1);
  // acks: the receiver has released the slot of epoch e - 2
  if (threadIdx.x < X.n) {
    const unsigned long long* ack =
        reinterpret_cast<const unsigned long long*>(P.base[me] + flags_off) + world + X.peer[threadIdx.x];
    if (e > 2) wait_geq(ack, e - 2);
  }
  __syncthreads();
  T* dst[kMaxXfer];
  for (int j = 0; j < X.n; ++j)
    dst[j] = reinterpret_cast<T*>(P.base[X.peer[j]] + slot_level_off +
                                  (size_t(par) * world + me) * slot_bytes);
  copy_ranges<T>(X, vec, dst, false);
  if (last_block(arrive) && threadIdx.x < X.n) {
    unsigned long long* f =
        reinterpret_cast<unsigned long long*>(P.base[X.peer[threadIdx.x]] + flags_off) + me;
    st_rel_sys(f, e);
  }
}

// halo pull: wait for every source, copy its slot into my ghost planes, ack
template <class T>
__device__ __forceinline__ void halo_pull(const Xfer& X, T* __restrict__ vec, const PeerPtrs& P, int me,
                                 size_t slot_level_off, size_t slot_bytes, int world,
                                 size_t flags_off, unsigned long long* ep, unsigned* arrive) {
  const unsigned long long e = ep[CH_HALO] + 1;
  const int par = int(e & 1);
  const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(P.base[me] + flags_off);
  if (threadIdx.x < X.n) wait_geq(fl + X.peer[threadIdx.x], e);
  __syncthreads();
  for (long long i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < X.total;
       i += int64_t(gridDim.x) * blockDim.x) {
    long long k = i;
    int j = 0;
    while (k >= X.count[j]) k -= X.count[j++];
    const T* slot = reinterpret_cast<const T*>(P.base[me] + slot_level_off +
                                               (size_t(par) * world + X.peer[j]) * slot_bytes);
    vec[X.dst_off[j] + k] = __ldcg(slot + X.src_off[j] + k);
  }
  if (last_block(arrive)) {
    if (threadIdx.x < X.n) {
      unsigned long long* ack = reinterpret_cast<unsigned long long*>(P.base[X.peer[threadIdx.x]] +
                                                                      flags_off) + world + me;
      st_rel_sys(ack, e);
    }
    if (threadIdx.x == 0) ep[CH_HALO] = e;
  }
}

// rank-ordered allreduce of n <= 8 doubles (one warp)
__global__ void peer_sum_kernel(double* vals, int n, PeerPtrs P, int me, int world, size_t sum_off,
                                size_t flags_off, unsigned long long* ep) {
  const unsigned long long e = ep[CH_SUM] + 1;
  const int par = int(e & 1);
  const int lane = threadIdx.x;
  for (int r = lane; r < world; r += 32) {
    double* slot = reinterpret_cast<double*>(P.base[r] + sum_off) + (size_t(par) * world + me) * kSumMax;
    for (int k = 0; k < n; ++k) slot[k] = vals[k];
  }
  __threadfence_system();
  __syncwarp();
  for (int r = lane; r < world; r += 32)
    st_rel_sys(reinterpret_cast<unsigned long long*>(P.base[r] + flags_off) + 2 * world + me, e);
  const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(P.base[me] + flags_off) + 2 * world;
  for (int r = lane; r < world; r += 32) wait_geq(fl + r, e);
  __syncwarp();
  if (lane == 0) {
    const double* sl = reinterpret_cast<const double*>(P.base[me] + sum_off) + size_t(par) * world * kSumMax;
    for (int k = 0; k < n; ++k) {
      double acc = __ldcg(sl + k);
      for (int r = 1; r < world; ++r) acc += __ldcg(sl + size_t(r) * kSumMax + k);
      vals[k] = acc;
    }
    ep[CH_SUM] = e;
  }
}

// allgather push: my owned planes -> every rank's gather slot (same offset)
__device__ __forceinline__ void gather_push(const double* __restrict__ win, long long src_off, long long dst_off,
                                   long long count, const PeerPtrs& P, int me, int world, size_t gather_off,
                                   size_t gather_bytes, size_t flags_off, unsigned long long* ep,
                                   unsigned* arrive) {
  const unsigned long long e = ep[CH_GATHER] + 1;
  const int par = int(e & 1);
  for (long long i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double v = win[src_off + i];
    for (int r = 0; r < world; ++r)
      reinterpret_cast<double*>(P.base[r] + gather_off + size_t(par) * gather_bytes)[dst_off + i] = v;
  }
  if (last_block(arrive))
    for (int r = threadIdx.x; r < world; r += blockDim.x)
      st_rel_sys(reinterpret_cast<unsigned long long*>(P.base[r] + flags_off) + 3 * world + me, e);
}

__device__ __forceinline__ void gather_pull(double* __restrict__ full, long long n, const PeerPtrs& P, int me,
                                   int world, size_t gather_off, size_t gather_bytes,
                                   size_t flags_off, unsigned long long* ep, unsigned* arrive) {
  const unsigned long long e = ep[CH_GATHER] + 1;
  const int par = int(e & 1);
  const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(P.base[me] + flags_off) + 3 * world;
  for (int r = threadIdx.x; r < world; r += blockDim.x) wait_geq(fl + r, e);
  __syncthreads();
  const double* sl = reinterpret_cast<const double*>(P.base[me] + gather_off + size_t(par) * gather_bytes);
  for (long long i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    full[i] = __ldcg(sl + i);
  if (last_block(arrive) && threadIdx.x == 0) ep[CH_GATHER] = e;
}

// One launch per exchange: the push, then (every block, once its own part is
// stored) the wait for the peers' flags and the pull.  Blocks that finished
// pushing spin on peer flags, so the grid must be co-resident: at most one
// block per SM (xfer_blocks).  The epoch is read by every block before the last
// block of the pull advances it (that block is last only after all arrived).
template <class T>
__global__ void halo_xchg_kernel(Xfer S, Xfer R, T* __restrict__ vec, PeerPtrs P, int me,
                                 size_t slot_level_off, size_t slot_bytes, int world,
                                 size_t flags_off, unsigned long long* ep, unsigned* arrive) {
  halo_push<T>(S, vec, P, me, slot_level_off, slot_bytes, world, flags_off, ep, arrive);
  halo_pull<T>(R, vec, P, me, slot_level_off, slot_bytes, world, flags_off, ep, arrive + 1);
}
__global__ void gather_xchg_kernel(const double* __restrict__ win, long long src_off, long long dst_off,
                                   long long count, double* __restrict__ full, long long nfull,
                                   PeerPtrs P, int me, int world, size_t gather_off,
                                   size_t gather_bytes, size_t flags_off, unsigned long long* ep,
                                   unsigned* arrive) {
  gather_push(win, src_off, dst_off, count, P, me, world, gather_off, gather_bytes, flags_off, ep, arrive);
  gather_pull(full, nfull, P, me, world, gather_off, gather_bytes, flags_off, ep, arrive + 1);
}

int xfer_blocks(long long n) {
  return int(std::max<long long>(1, std::min<long long>((n + 255) / 256, num_sms())));
}

}  // namespace

// Ghost transfers of one level, (src, dst, p0, p1) in (dst, plane) order:
// slab.py halo_pieces, restated here so both sides derive the same list.
std::vector<std::array<int, 4>> halo_pieces(const std::vector<std::array<int, 4>>& win) {
  std::vector<std::array<int, 4>> out;
  auto owner = [&](int p) {
    for (size_t r = 0; r < win.size(); ++r)
      if (win[r][2] <= p && p < win[r][3]) return int(r);
    throw Error("plane without owner in the slab plan");
  };
  for (size_t dst = 0; dst < win.size(); ++dst) {
    const auto& w = win[dst];
    const int rng[2][2] = {{w[0], w[2]}, {w[3], w[1] + 1}};
    for (auto& lh : rng) {
      int p = lh[0];
      while (p < lh[1]) {
        const int src = owner(p);
        const int q = std::min(lh[1], win[size_t(src)][3]);
        SG_REQUIRE(src != int(dst), "ghost plane owned by its own rank");
        out.push_back({src, int(dst), p, q});
        p = q;
      }
    }
  }
  return out;
}

struct PeerComm {
  int rank = 0, world = 1, n_dist = 0;
  // exchange levels: 0, 1 = slab levels (node layout), kP32Level = level 0 in
  // the P32 layout (same planes as level 0, 3 XS (ny+1) floats each)
  std::vector<std::array<int, 4>> win[3];  // [level][rank] = {w0, w1, o0, o1}
  int64_t pnd[3] = {0, 0, 0};              // elements per node plane (0: level unused)
  int full_planes[3] = {0, 0, 0};
  size_t off_halo[3] = {0, 0, 0}, slot_bytes[3] = {0, 0, 0};
  size_t off_sum = 0, off_gather = 0, gather_bytes = 0, off_flags = 0, total = 0;
  char* base = nullptr;
  PeerPtrs P{};
  std::vector<bool> opened;  // peer mapped through cudaIpcOpenMemHandle
  DBuf<unsigned long long> ep;
  DBuf<unsigned> arrive;
  Xfer push[3], pull[3];  // per exchange level (element counts, any width)

  ~PeerComm() {
    for (int r = 0; r < world; ++r)
      if (r < int(opened.size()) && opened[size_t(r)] && P.base[r]) cudaIpcCloseMemHandle(P.base[r]);
    if (base) cudaFree(base);
  }

  static size_t up(size_t v) { return (v + 255) & ~size_t(255); }

  void setup(int rank_, int world_, int n_dist_, const int* planes_all, const int64_t* pnd_,
             const int* full_planes_, int64_t p32_plane, cudaStream_t s) {
    SG_REQUIRE(world_ >= 1 && world_ <= kMaxRanks, "peer transport: 1..64 ranks");
    rank = rank_;
    world = world_;
    n_dist = n_dist_;
    for (int l = 0; l < n_dist; ++l) {
      pnd[l] = pnd_[l];
      full_planes[l] = full_planes_[l];
      win[l].resize(size_t(world));
      for (int r = 0; r < world; ++r)
        for (int k = 0; k < 4; ++k) win[l][size_t(r)][size_t(k)] = planes_all[(r * n_dist + l) * 4 + k];
    }
    if (p32_plane > 0) {
      pnd[kP32Level] = p32_plane;
      win[kP32Level] = win[0];
    }
    size_t off = 0;
    for (int l = 0; l < 3; ++l) {
      if (!pnd[l]) continue;
      int maxg = 0;
      for (auto& w : win[l]) maxg = std::max(maxg, (w[2] - w[0]) + (w[1] + 1 - w[3]));
      slot_bytes[l] = up(size_t(std::max(maxg, 1)) * size_t(pnd[l]) * (l == kP32Level ? 4 : 8));
      off_halo[l] = off;
      off += 2 * size_t(world) * slot_bytes[l];
    }
    off_sum = off;
    off += up(2 * size_t(world) * kSumMax * 8);
    // gathers run at the cut level (dist_level) and on level 0 (API boundary)
    gather_bytes = 0;
    for (int l = 0; l < n_dist; ++l)
      gather_bytes = std::max(gather_bytes, up(size_t(full_planes[l]) * size_t(pnd[l]) * 8));
    off_gather = off;
    off += 2 * gather_bytes;
    off_flags = off;
    off += up(4 * size_t(world) * 8);
    total = off;
    SG_CUDA(cudaMalloc(&base, total));
    SG_CUDA(cudaMemsetAsync(base + off_flags, 0, total - off_flags, s));
    ep.alloc(4);
    ep.zero(s);
    arrive.alloc(4);
    SG_CUDA(cudaMemsetAsync(arrive.p, 0, 4 * sizeof(unsigned), s));
    SG_CUDA(cudaStreamSynchronize(s));
    opened.assign(size_t(world), false);
    P.base[rank] = base;
    // transfer lists of this rank (element offsets for 8- and 4-byte vectors)
    for (int l = 0; l < 3; ++l) {
      if (!pnd[l]) continue;
      const auto pcs = halo_pieces(win[l]);
      {
        const int64_t epp = pnd[l];  // elements per plane (8- or 4-byte elements alike)
        Xfer& ps = push[l];
        Xfer& pl = pull[l];
        ps = Xfer{};
        pl = Xfer{};
        for (auto& pc : pcs) {
          const int src = pc[0], dst = pc[1], p0 = pc[2], p1 = pc[3];
          const long long cnt = (long long)(p1 - p0) * epp;
          if (src == rank) {
            SG_REQUIRE(ps.n < kMaxXfer, "too many halo sends");
            ps.peer[ps.n] = dst;
            ps.src_off[ps.n] = (long long)(p0 - win[l][size_t(rank)][0]) * epp;
            ps.dst_off[ps.n] = 0;
            ps.count[ps.n] = cnt;
            ps.total += cnt;
            ++ps.n;
          }
          if (dst == rank) {
            SG_REQUIRE(pl.n < kMaxXfer, "too many halo receives");
            pl.peer[pl.n] = src;
            pl.src_off[pl.n] = 0;
            pl.dst_off[pl.n] = (long long)(p0 - win[l][size_t(rank)][0]) * epp;
            pl.count[pl.n] = cnt;
            pl.total += cnt;
            ++pl.n;
          }
        }
      }
    }
  }

  void open(const char* handles, const unsigned long long* ptrs) {
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      if (ptrs) {
        P.base[r] = reinterpret_cast<char*>(ptrs[r]);
      } else {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + size_t(r) * sizeof(cudaIpcMemHandle_t), sizeof(h));
        void* p = nullptr;
        SG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        P.base[r] = static_cast<char*>(p);
        opened[size_t(r)] = true;
      }
    }
  }

  void halo(int level, void* vec, int eb, cudaStream_t s) {
    SG_REQUIRE(level >= 0 && level < 3 && pnd[level] && (eb == 8 || eb == 4) &&
                   (level != kP32Level || eb == 4), "bad halo request");
    if (world == 1) return;  // no ghost planes: nothing to move
    const Xfer& ps = push[level];
    const Xfer& pl = pull[level];
    const long long nmax = std::max(ps.total, pl.total);
    if (eb == 8)
      halo_xchg_kernel<unsigned long long><<<xfer_blocks(nmax), 256, 0, s>>>(
          ps, pl, static_cast<unsigned long long*>(vec), P, rank, off_halo[level], slot_bytes[level],
          world, off_flags, ep.p, arrive.p);
    else
      halo_xchg_kernel<unsigned><<<xfer_blocks(nmax), 256, 0, s>>>(
          ps, pl, static_cast<unsigned*>(vec), P, rank, off_halo[level], slot_bytes[level], world,
          off_flags, ep.p, arrive.p);
    SG_CHECK_LAUNCH();
  }

  void sum(double* vals, int n, cudaStream_t s) {
    SG_REQUIRE(n >= 1 && n <= kSumMax, "peer allreduce: 1..8 values");
    if (world == 1) return;  // the rank-ordered sum of one value is the value
    peer_sum_kernel<<<1, 32, 0, s>>>(vals, n, P, rank, world, off_sum, off_flags, ep.p);
    SG_CHECK_LAUNCH();
  }

  void gather(int level, const double* win_vec, double* full, cudaStream_t s) {
    SG_REQUIRE(level == n_dist - 1 || level == 0, "gather of a slab level");
    const auto& w = win[level][size_t(rank)];
    const long long cnt = (long long)(w[3] - w[2]) * pnd[level];
    const long long src = (long long)(w[2] - w[0]) * pnd[level];
    const long long dst = (long long)w[2] * pnd[level];
    const long long nfull = (long long)full_planes[level] * pnd[level];
    SG_REQUIRE(size_t(nfull) * 8 <= gather_bytes, "gather slot too small for this level");
    if (world == 1) {  // the window is the whole level
      SG_CUDA(cudaMemcpyAsync(full + dst, win_vec + src, size_t(cnt) * 8, cudaMemcpyDeviceToDevice, s));
      return;
    }
    gather_xchg_kernel<<<xfer_blocks(std::max(cnt, nfull)), 256, 0, s>>>(
        win_vec, src, dst, cnt, full, nfull, P, rank, world, off_gather, gather_bytes, off_flags,
        ep.p, arrive.p + 2);
    SG_CHECK_LAUNCH();
  }
};

namespace {
// the hooks cross a C function-pointer boundary: report failures by status,
// with the reason on stderr (CommHooks then raises "slab ... failed")
template <class F>
int hook_call(const char* what, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    fprintf(stderr, "peer transport %s: %s\n", what, e.what());
  } catch (...) {
    fprintf(stderr, "peer transport %s: unknown error\n", what);
  }
  return 1;
}
int hook_halo(void* ctx, int level, void* vec, int eb, void* stream) {
  return hook_call("halo", [&] {
    static_cast<PeerComm*>(ctx)->halo(level, vec, eb, static_cast<cudaStream_t>(stream));
  });
}
int hook_sum(void* ctx, double* vals, int n, void* stream) {
  return hook_call("sum", [&] {
    static_cast<PeerComm*>(ctx)->sum(vals, n, static_cast<cudaStream_t>(stream));
  });
}
int hook_gather(void* ctx, int level, const double* win, double* full, void* stream) {
  return hook_call("gather", [&] {
    static_cast<PeerComm*>(ctx)->gather(level, win, full, static_cast<cudaStream_t>(stream));
  });
}
}  // namespace

PeerComm* peer_create(int rank, int world, int n_dist, const int* planes_all, const int64_t* pnd,
                      const int* full_planes, int64_t p32_plane, cudaStream_t s, CommHooks& hooks) {
  auto pc = std::make_unique<PeerComm>();
  pc->setup(rank, world, n_dist, planes_all, pnd, full_planes, p32_plane, s);
  hooks.ctx = pc.get();
  hooks.halo = hook_halo;
  hooks.allreduce = hook_sum;
  hooks.allgather = hook_gather;
  return pc.release();
}
void peer_destroy(PeerComm* p) { delete p; }
void peer_handle(PeerComm* p, void* out) {
  cudaIpcMemHandle_t h;
  SG_CUDA(cudaIpcGetMemHandle(&h, p->base));
  std::memcpy(out, &h, sizeof(h));
}
unsigned long long peer_base(PeerComm* p) { return reinterpret_cast<unsigned long long>(p->base); }
bool peer_sum_dev(const PeerComm* p, PeerSumDev& out) {
  if (!p) return false;
  for (int r = 0; r < kPeerMaxRanks; ++r) out.base[r] = r < p->world ? p->P.base[r] : nullptr;
  out.me = p->rank;
  out.world = p->world;
  out.sum_off = p->off_sum;
  out.flags_off = p->off_flags;
  out.ep = p->ep.p;
  return true;
}
void peer_open(PeerComm* p, const void* handles, const unsigned long long* ptrs) {
  p->open(static_cast<const char*>(handles), ptrs);
}

}  // namespace sg
