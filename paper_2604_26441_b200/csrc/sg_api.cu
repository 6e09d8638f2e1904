// extern "C" boundary (include/sg_api.h).  Every entry point catches C++
// exceptions and CUDA errors and turns them into a nonzero status plus a
// thread-local message; nothing throws across the ABI.
#include <cstring>
#include <mutex>
#include "../../include/sg_api.h"
#include "sg_hier.cuh"

struct sg_fine {
  sg::FineOp op;
  sg::FineWork w;
  std::mutex mu;
};

struct sg_hier {
  sg_fine* fine = nullptr;
  std::unique_ptr<sg::Hier> h;
  std::mutex mu;
};

struct sg_dist {
  sg_hier* hier = nullptr;
  std::unique_ptr<sg::DistPart> d;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
  } catch (...) {
    g_err = "unknown error";
  }
  return 1;
}

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

sg::Level& level_of(sg_hier* h, int level) {
  SG_REQUIRE(!h->h->released, "hierarchy levels were released to a slab solver");
  SG_REQUIRE(level >= 0 && level < int(h->h->lv.size()), "level index out of range");
  return *h->h->lv[size_t(level)];
}

// free-layout staging buffers for level-wise API calls
struct Stage {
  sg::DBuf<double> a, b;
  sg::DBuf<float> fa, fb;
  explicit Stage(int64_t nd) : a(static_cast<size_t>(nd)), b(static_cast<size_t>(nd)) {}
};

}  // namespace

extern "C" {

const char* sg_last_error(void) { return g_err.c_str(); }
int sg_version(void) { return 1; }

// ---------------------------------------------------------------- fine
int sg_fine_create(int nx, int ny, int nz, const uint8_t* dof_mask, const double* E,
                   const double* ke, sg_fine** out) {
  return guard([&] {
    SG_REQUIRE(out && E && ke, "null argument");
    auto f = std::make_unique<sg_fine>();
    cudaStream_t s = 0;
    sg::build_grid(f->op.grid, nx, ny, nz, dof_mask, s);
    const int64_t ne = f->op.grid.d.nelem();
    std::vector<float> e32(static_cast<size_t>(ne));
    double emax = -INFINITY;
    for (int64_t e = 0; e < ne; ++e) {
      e32[size_t(e)] = float(E[e]);
      emax = E[e] > emax ? E[e] : emax;
    }
    f->op.emax = emax;
    f->op.E64.alloc(size_t(ne));
    f->op.E64.upload(E, size_t(ne), s);
    f->op.E32.alloc(size_t(ne));
    f->op.E32.upload(e32.data(), size_t(ne), s);
    std::memcpy(f->op.ke_host, ke, sizeof(double) * 576);
    for (int q = 0; q < 576; ++q) {
      f->op.ke64.k[q] = ke[q];
      f->op.ke32.k[q] = float(ke[q]);
      f->op.ke16.k[q] = sg::bf16_round(float(ke[q]));
    }
    for (int q = 0; q < 24; ++q) f->op.kdiag.d[q] = ke[q * 24 + q];
    f->op.walsh_ok = sg::walsh_params(ke, f->op.kw64, f->op.kw32);
    if (sg::p32_supported(f->op)) {  // P32 staging of the node-layout FP32 apply
      const size_t n32 = size_t(sg::p32_size(f->op.grid.d));
      f->op.p32a.alloc(n32);
      f->op.p32b.alloc(n32);
      f->op.p32a.zero(s);
      f->op.p32b.zero(s);
    }
    const size_t nd = size_t(3 * f->op.grid.d.nnodes());
    f->w.u64.alloc(nd);
    f->w.y64.alloc(nd);
    f->w.u32.alloc(nd);
    f->w.y32.alloc(nd);
    f->w.scal.alloc(8);
    SG_CUDA(cudaStreamSynchronize(s));
    *out = f.release();
  });
}

void sg_fine_destroy(sg_fine* op) { delete op; }

int64_t sg_fine_n_free(const sg_fine* op) { return op ? op->op.grid.n_free : -1; }

int sg_fine_apply(sg_fine* f, int tag, const void* u, void* y, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    cudaStream_t s = S(stream);
    if (tag == SG_TAG_FP64) {
      sg::scatter_free<double>(f->op.grid, (const double*)u, f->w.u64.p, s);
      sg::fine_apply_f64(f->op, f->w.u64.p, f->w.y64.p, s);
      sg::gather_free<double>(f->op.grid, f->w.y64.p, (double*)y, s);
    } else {
      sg::scatter_free<float>(f->op.grid, (const float*)u, f->w.u32.p, s);
      sg::fine_apply_tag(f->op, tag, f->w.u32.p, f->w.y32.p, s);
      sg::gather_free<float>(f->op.grid, f->w.y32.p, (float*)y, s);
    }
  });
}

int sg_fine_diagonal(sg_fine* f, double* d, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    sg::fine_floored_diag(f->op, f->w, S(stream));
    sg::gather_free<double>(f->op.grid, f->w.diag.p, d, S(stream));
  });
}

int sg_fine_dense(sg_fine* f, double* K, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    cudaStream_t s = S(stream);
    SG_REQUIRE(f->op.grid.n_free <= 20000, "dense assembly limited to 20000 free DOFs");
    sg::DBuf<double> A(static_cast<size_t>(243 * f->op.grid.d.nnodes()));
    sg::fine_to_stencil(f->op, A.p, s);
    sg::stencil_to_dense(f->op.grid, A.p, K, 0.0, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_fine_boundary_codes(sg_fine* f, uint32_t* codes, int cap, int* n) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    std::vector<uint32_t> c;
    sg::boundary_codes(f->op, c, 0);
    *n = int(c.size());
    if (codes == nullptr) return;  // size query
    SG_REQUIRE(int(c.size()) <= cap, "boundary code buffer too small");
    std::copy(c.begin(), c.end(), codes);
  });
}

// ----------------------------------------------------------- hierarchy
int sg_hier_create(sg_fine* f, const sg_hier_params* p, const double* triples,
                   const uint32_t* codes, const double* diffs, int ncodes,
                   const double* lam_cache, int n_cache, void* stream, sg_hier** out) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    SG_REQUIRE(p && triples && out, "null argument");
    sg::HParams hp;
    hp.levels = p->levels;
    hp.policy = p->policy;
    hp.smoother_kind = p->smoother_kind;
    hp.degree = p->degree;
    hp.alpha = p->alpha;
    hp.omega = p->omega;
    hp.coarse_smooth_steps = p->coarse_smooth_steps;
    hp.cholesky_cutoff = p->cholesky_cutoff;
    hp.coarse_pcg_steps = p->coarse_pcg_steps;
    hp.power_seed = p->power_seed;
    sg::L1Tables t;
    std::memcpy(t.tri, triples, sizeof(double) * 8 * 576);
    t.codes.assign(codes, codes + ncodes);
    t.diffs.assign(diffs, diffs + size_t(ncodes) * 576);
    auto h = std::make_unique<sg_hier>();
    h->fine = f;
    h->h = sg::hier_build(&f->op, f->w, hp, t, lam_cache, n_cache, S(stream));
    *out = h.release();
  });
}

void sg_hier_destroy(sg_hier* h) { delete h; }

int sg_hier_get_info(sg_hier* h, sg_hier_info* info) {
  return guard([&] {
    info->n_levels = int(h->h->lv.size());
    info->clamped = h->h->clamped ? 1 : 0;
    info->coarsest_dense = h->h->coarsest_mode == 0 ? 1 : 0;
    info->eps = h->h->eps;
  });
}

int sg_hier_level_info(sg_hier* h, int level, sg_level_info* info) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    sg::Level& L = level_of(h, level);
    info->nx = L.g->d.nx;
    info->ny = L.g->d.ny;
    info->nz = L.g->d.nz;
    info->tag = L.tag;
    info->n_free = L.g->n_free;
    if (!L.is_fine && L.st.nnz == 0) L.st.nnz = sg::stencil_count_nnz(*L.g, L.st.A64.p, 0);
    info->nnz = L.is_fine ? 0 : L.st.nnz;
    info->lam_max = L.lam;
  });
}

int sg_hier_level_csr(sg_hier* h, int level, int64_t* indptr, int64_t* indices, double* data) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    sg::Level& L = level_of(h, level);
    SG_REQUIRE(!L.is_fine, "level 0 is matrix-free");
    sg::stencil_export_csr(*L.g, L.st.A64.p, indptr, indices, data, 0);
  });
}

int sg_hier_level_mask(sg_hier* h, int level, uint8_t* mask) {
  return guard([&] {
    sg::Level& L = level_of(h, level);
    const int64_t nn = L.g->d.nnodes();
    for (int64_t n = 0; n < nn; ++n)
      for (int a = 0; a < 3; ++a) mask[3 * n + a] = (L.g->h_nmask[size_t(n)] >> a) & 1;
  });
}

int sg_hier_level_diag(sg_hier* h, int level, double* d, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    sg::Level& L = level_of(h, level);
    sg::gather_free<double>(*L.g, L.diag.p, d, S(stream));
  });
}

int sg_hier_cycle(sg_hier* h, int gamma, const double* r, double* z, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    SG_REQUIRE(!h->h->released, "hierarchy levels were released to a slab solver (single-GPU cycle unavailable)");
    cudaStream_t s = S(stream);
    sg::Level& L0 = *h->h->lv[0];
    sg::scatter_free<double>(*L0.g, r, L0.w.r.p, s);
    sg::cycle_run(*h->h, gamma, s);
    sg::gather_free<double>(*L0.g, L0.w.x.p, z, s);
  });
}

int sg_hier_level_apply(sg_hier* h, int level, int tag, const void* x, void* y, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    sg::Level& L = level_of(h, level);
    const int64_t nd = L.nd();
    Stage st(nd);
    if (tag == SG_TAG_FP64) {
      sg::scatter_free<double>(*L.g, (const double*)x, st.a.p, s);
      sg::level_apply(*h->h, L, tag, st.a.p, st.b.p, s);
      sg::gather_free<double>(*L.g, st.b.p, (double*)y, s);
    } else {
      st.fa.alloc(size_t(nd));
      st.fb.alloc(size_t(nd));
      sg::scatter_free<float>(*L.g, (const float*)x, st.fa.p, s);
      sg::level_apply(*h->h, L, tag, st.fa.p, st.fb.p, s);
      sg::gather_free<float>(*L.g, st.fb.p, (float*)y, s);
    }
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_hier_level_smooth(sg_hier* h, int level, const double* b, const double* x0, double* out,
                         void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    sg::Level& L = level_of(h, level);
    const int64_t nd = L.nd();
    Stage st(nd);
    sg::DBuf<double> xo(static_cast<size_t>(nd));
    sg::scatter_free<double>(*L.g, b, st.a.p, s);
    if (x0) sg::scatter_free<double>(*L.g, x0, st.b.p, s);
    sg::level_smooth(*h->h, level, st.a.p, x0 ? st.b.p : nullptr, xo.p, s);
    sg::gather_free<double>(*L.g, xo.p, out, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_hier_prolong(sg_hier* h, int level, const double* xc, double* xf, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    SG_REQUIRE(level + 1 < int(h->h->lv.size()), "no coarser level");
    sg::Level& F = level_of(h, level);
    sg::Level& C = level_of(h, level + 1);
    sg::DBuf<double> a(static_cast<size_t>(C.nd())), b(static_cast<size_t>(F.nd()));
    sg::scatter_free<double>(*C.g, xc, a.p, s);
    sg::prolong(*F.g, *C.g, a.p, b.p, false, s);
    sg::gather_free<double>(*F.g, b.p, xf, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_hier_restrict(sg_hier* h, int level, const double* xf, double* xc, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    SG_REQUIRE(level + 1 < int(h->h->lv.size()), "no coarser level");
    sg::Level& F = level_of(h, level);
    sg::Level& C = level_of(h, level + 1);
    sg::DBuf<double> a(static_cast<size_t>(F.nd())), b(static_cast<size_t>(C.nd()));
    sg::scatter_free<double>(*F.g, xf, a.p, s);
    sg::restrict_(*F.g, *C.g, a.p, b.p, s);
    sg::gather_free<double>(*C.g, b.p, xc, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_hier_coarsest_solve(sg_hier* h, const double* r, double* x, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    sg::Level& L = *h->h->lv.back();
    sg::scatter_free<double>(*L.g, r, L.w.r.p, s);
    sg::coarsest_solve(*h->h, L.w.r.p, L.w.x.p, s);
    sg::gather_free<double>(*L.g, L.w.x.p, x, s);
  });
}

int sg_hier_transfer_csr(sg_hier* h, int level, int64_t* indptr, int64_t* indices, double* data,
                         int64_t* nnz) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    SG_REQUIRE(level + 1 < int(h->h->lv.size()), "no coarser level");
    sg::transfer_export_csr(*level_of(h, level).g, *level_of(h, level + 1).g, indptr, indices,
                            data, nnz, 0);
  });
}

// -------------------------------------------------------------- solvers
static int run_solver(int which, sg_fine* f, int ktag, sg_hier* h, int gamma, const double* b,
                      double* x, const sg_solver_cfg* cfg, sg_report* rep, double* history,
                      void* stream) {
  return guard([&] {
    std::unique_lock<std::mutex> lf(f->mu);
    std::unique_lock<std::mutex> lh;
    if (h) {
      SG_REQUIRE(h->fine == f, "hierarchy built for a different operator");
      SG_REQUIRE(!h->h->released, "hierarchy levels were released to a slab solver");
      lh = std::unique_lock<std::mutex>(h->mu);
    }
    cudaStream_t s = S(stream);
    sg::fine_floored_diag(f->op, f->w, s);
    sg::NativeSys sys{&f->op, &f->w, ktag, h ? h->h.get() : nullptr, gamma};
    sg::SolverCfg c{cfg->tol, cfg->maxiter, cfg->restart};
    sg::SolveOut o;
    std::vector<double> hist;
    const int64_t nd = 3 * f->op.grid.d.nnodes();
    struct {
      double* p;
    } bn{f->w.sw.vec(6, nd)}, xn{f->w.sw.vec(7, nd)};
    sg::scatter_free<double>(f->op.grid, b, bn.p, s);
    if (which == 0) sg::pcg_native(sys, bn.p, xn.p, c, o, hist, s);
    else sg::fgmres_native(sys, bn.p, xn.p, c, o, hist, s);
    sg::gather_free<double>(f->op.grid, xn.p, x, s);
    SG_CUDA(cudaStreamSynchronize(s));
    rep->converged = o.converged;
    rep->iterations = o.iterations;
    rep->final_true_residual = o.final_true_residual;
    rep->failure_kind = o.failure_kind;
    rep->wall_time = o.wall_time;
    if (history) std::copy(hist.begin(), hist.end(), history);
  });
}

int sg_pcg(sg_fine* f, int ktag, sg_hier* h, int gamma, const double* b, double* x,
           const sg_solver_cfg* cfg, sg_report* rep, double* history, void* stream) {
  return run_solver(0, f, ktag, h, gamma, b, x, cfg, rep, history, stream);
}

int sg_fgmres(sg_fine* f, int ktag, sg_hier* h, int gamma, const double* b, double* x,
              const sg_solver_cfg* cfg, sg_report* rep, double* history, void* stream) {
  return run_solver(1, f, ktag, h, gamma, b, x, cfg, rep, history, stream);
}

// ------------------------------------------------------- slab partition
int sg_dist_create(sg_hier* h, int n_dist, const int32_t* planes, const sg_comm* comm, void* stream,
                   sg_dist** out) {
  return guard([&] {
    SG_REQUIRE(h && planes && comm && out && comm->halo && comm->allreduce && comm->allgather,
               "null argument");
    SG_REQUIRE(!h->h->released, "hierarchy levels were released to a slab solver");
    std::lock_guard<std::mutex> lk(h->mu);
    sg::CommHooks c;
    c.ctx = comm->ctx;
    c.halo = comm->halo;
    c.allreduce = comm->allreduce;
    c.allgather = comm->allgather;
    std::vector<int> pl(planes, planes + 4 * n_dist);
    auto d = std::make_unique<sg_dist>();
    d->hier = h;
    d->d = sg::dist_build(*h->h, n_dist, pl.data(), c, S(stream));
    *out = d.release();
  });
}

int sg_dist_create_peer(sg_hier* h, int n_dist, const int32_t* planes_all, int rank, int world,
                        void* stream, sg_dist** out) {
  return guard([&] {
    SG_REQUIRE(h && planes_all && out && world >= 1 && rank >= 0 && rank < world, "bad argument");
    SG_REQUIRE(n_dist >= 1 && n_dist <= 2 && int(h->h->lv.size()) > n_dist, "1 or 2 slab levels");
    SG_REQUIRE(!h->h->released, "hierarchy levels were released to a slab solver");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    int64_t pnd[2] = {0, 0};
    int fpl[2] = {0, 0};
    for (int l = 0; l < n_dist; ++l) {
      const sg::GridDesc& g = h->h->lv[size_t(l)]->g->d;
      pnd[l] = 3 * int64_t(g.nx + 1) * (g.ny + 1);
      fpl[l] = g.nz + 1;
    }
    // level 0 in the P32 layout (FP32 level-0 smoother) exchanges its own planes
    const sg::Level& L0 = *h->h->lv[0];
    const int64_t p32_plane = L0.p32 ? 3 * int64_t(sg::p32_xs(L0.g->d)) * (L0.g->d.ny + 1) : 0;
    sg::CommHooks c;
    sg::PeerComm* pc = sg::peer_create(rank, world, n_dist, planes_all, pnd, fpl, p32_plane, s, c);
    std::vector<int> pl(planes_all + size_t(rank) * n_dist * 4, planes_all + size_t(rank + 1) * n_dist * 4);
    auto d = std::make_unique<sg_dist>();
    d->hier = h;
    try {
      d->d = sg::dist_build(*h->h, n_dist, pl.data(), c, s);
    } catch (...) {
      sg::peer_destroy(pc);
      throw;
    }
    d->d->peer = pc;
    *out = d.release();
  });
}

int sg_dist_peer_handle(sg_dist* d, void* handle_out, uint64_t* base_out) {
  return guard([&] {
    SG_REQUIRE(d && d->d->peer, "not a device-transport slab handle");
    if (handle_out) sg::peer_handle(d->d->peer, handle_out);
    if (base_out) *base_out = sg::peer_base(d->d->peer);
  });
}

int sg_dist_peer_open(sg_dist* d, const void* handles, const uint64_t* bases) {
  return guard([&] {
    SG_REQUIRE(d && d->d->peer && (handles || bases), "bad argument");
    sg::peer_open(d->d->peer, handles, reinterpret_cast<const unsigned long long*>(bases));
  });
}

int sg_dist_release_full(sg_dist* d, void* stream) {
  return guard([&] {
    SG_REQUIRE(d, "null argument");
    std::lock_guard<std::mutex> lk(d->hier->mu);
    sg::dist_release_full(*d->d, S(stream));
  });
}

int sg_plan_halo(int world, const int32_t* windows, int32_t* out, int cap) {
  return guard([&] {
    std::vector<std::array<int, 4>> w(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r)
      for (int k = 0; k < 4; ++k) w[size_t(r)][size_t(k)] = windows[4 * r + k];
    const auto pcs = sg::halo_pieces(w);
    SG_REQUIRE(int(pcs.size()) <= cap, "piece buffer too small");
    for (size_t i = 0; i < pcs.size(); ++i)
      for (int k = 0; k < 4; ++k) out[4 * i + size_t(k)] = pcs[i][size_t(k)];
    out[4 * pcs.size()] = -1;
  });
}

void sg_dist_destroy(sg_dist* d) { delete d; }

namespace {
// global free vector -> this rank's window (node layout)
void to_window(sg::DistPart& D, const double* x_free, double* xw, cudaStream_t s) {
  const sg::Grid& fg = D.full->fine->grid;
  sg::scatter_free<double>(fg, x_free, D.bfull.p, s);
  SG_CUDA(cudaMemcpyAsync(xw, D.bfull.p + int64_t(D.w0[0]) * D.plane_nd(0),
                          sizeof(double) * D.W->lv[0]->nd(), cudaMemcpyDeviceToDevice, s));
}
// owned planes of every rank -> global free vector
void from_window(sg::DistPart& D, const double* yw, double* y_free, cudaStream_t s) {
  D.comm.gather(0, yw, D.xfull.p, s);
  sg::gather_free<double>(D.full->fine->grid, D.xfull.p, y_free, s);
}
}  // namespace

int sg_dist_solve(sg_dist* dd, int method, int ktag, int gamma, const double* b, double* x,
                  const sg_solver_cfg* cfg, sg_report* rep, double* history, void* stream) {
  return guard([&] {
    SG_REQUIRE(dd && cfg && rep, "null argument");
    std::unique_lock<std::mutex> lf(dd->hier->fine->mu);
    std::unique_lock<std::mutex> lh(dd->hier->mu);
    sg::DistPart& D = *dd->d;
    cudaStream_t s = S(stream);
    sg::NativeSys sys{&D.wfine, &D.wfw, ktag, D.W.get(), gamma, &D};
    sg::SolverCfg c{cfg->tol, cfg->maxiter, cfg->restart};
    sg::SolveOut o;
    std::vector<double> hist;
    const int64_t nd = D.W->lv[0]->nd();
    double* bw = D.wfw.sw.vec(6, nd);
    double* xw = D.wfw.sw.vec(7, nd);
    to_window(D, b, bw, s);
    if (method == 0) sg::pcg_native(sys, bw, xw, c, o, hist, s);
    else sg::fgmres_native(sys, bw, xw, c, o, hist, s);
    from_window(D, xw, x, s);
    SG_CUDA(cudaStreamSynchronize(s));
    rep->converged = o.converged;
    rep->iterations = o.iterations;
    rep->final_true_residual = o.final_true_residual;
    rep->failure_kind = o.failure_kind;
    rep->wall_time = o.wall_time;
    if (history) std::copy(hist.begin(), hist.end(), history);
  });
}

int sg_dist_apply(sg_dist* dd, int what, int ktag, int gamma, const double* x, double* y,
                  void* stream) {
  return guard([&] {
    SG_REQUIRE(dd && x && y, "null argument");
    std::unique_lock<std::mutex> lf(dd->hier->fine->mu);
    std::unique_lock<std::mutex> lh(dd->hier->mu);
    sg::DistPart& D = *dd->d;
    cudaStream_t s = S(stream);
    sg::NativeSys sys{&D.wfine, &D.wfw, ktag, D.W.get(), gamma, &D};
    const int64_t nd = D.W->lv[0]->nd();
    double* xw = D.wfw.sw.vec(4, nd);
    double* yw = D.wfw.sw.vec(5, nd);
    to_window(D, x, xw, s);
    sg::dist_apply(sys, what, xw, yw, s);
    from_window(D, yw, y, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_lanczos(sg_fine* f, sg_hier* h, int gamma, int m, uint64_t seed, double* H, int* used,
               int* partial, void* stream) {
  return guard([&] {
    std::unique_lock<std::mutex> lf(f->mu);
    std::unique_lock<std::mutex> lh(h->mu);
    SG_REQUIRE(h->fine == f, "hierarchy built for a different operator");
    sg::NativeSys sys{&f->op, &f->w, SG_TAG_FP64, h->h.get(), gamma};
    std::vector<double> Hv;
    int u = 0;
    bool part = false;
    sg::lanczos_native(sys, m, seed, Hv, u, part, S(stream));
    std::copy(Hv.begin(), Hv.end(), H);
    *used = u;
    *partial = part ? 1 : 0;
  });
}

}  // extern "C"

// ------------------------------------------------------------ vectors
namespace {

template <class T>
struct DotT {
  const T* a;
  const T* b;
  __device__ void operator()(int64_t i, double (&acc)[1]) const {
    acc[0] += double(a[i]) * double(b[i]);
  }
};

template <class T> __device__ __forceinline__ T mulr(T a, T b);
template <> __device__ __forceinline__ double mulr(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mulr(float a, float b) { return __fmul_rn(a, b); }
template <class T> __device__ __forceinline__ T addr(T a, T b);
template <> __device__ __forceinline__ double addr(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float addr(float a, float b) { return __fadd_rn(a, b); }
template <class T> __device__ __forceinline__ T subr(T a, T b);
template <> __device__ __forceinline__ double subr(double a, double b) { return __dsub_rn(a, b); }
template <> __device__ __forceinline__ float subr(float a, float b) { return __fsub_rn(a, b); }
template <class T> __device__ __forceinline__ T divr(T a, T b);
template <> __device__ __forceinline__ double divr(double a, double b) { return __ddiv_rn(a, b); }
template <> __device__ __forceinline__ float divr(float a, float b) { return __fdiv_rn(a, b); }

// op: 0 axpy (y = y + s*x), 1 xpby (y = x + s*y), 2 sub (c = a - b), 3 mul, 4 scale, 5 div
template <class T>
__global__ void vec_kernel(int op, int64_t n, const T* __restrict__ a, const T* __restrict__ b,
                           T* __restrict__ c, T sc) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  switch (op) {
    case 0: c[i] = addr(c[i], mulr(sc, a[i])); break;
    case 1: c[i] = addr(a[i], mulr(sc, c[i])); break;
    case 2: c[i] = subr(a[i], b[i]); break;
    case 3: c[i] = mulr(a[i], b[i]); break;
    case 4: c[i] = mulr(a[i], sc); break;
    case 5: c[i] = divr(a[i], sc); break;
  }
}

__global__ void bf16_kernel(int64_t n, const float* __restrict__ a, float* __restrict__ b) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = sg::bf16_round(a[i]);
}

thread_local sg::RedWork t_red;
thread_local sg::DBuf<double> t_scal;

int vec_op(int dtype, int op, int64_t n, const void* a, const void* b, void* c, double sc,
           void* stream) {
  return guard([&] {
    if (n <= 0) return;
    const int nb = sg::grid_blocks(n, 256);
    if (dtype == 0)
      vec_kernel<double><<<nb, 256, 0, S(stream)>>>(op, n, (const double*)a, (const double*)b,
                                                     (double*)c, sc);
    else
      vec_kernel<float><<<nb, 256, 0, S(stream)>>>(op, n, (const float*)a, (const float*)b,
                                                    (float*)c, float(sc));
    SG_CHECK_LAUNCH();
  });
}

}  // namespace

extern "C" {

int sg_vec_dot(int dtype, int64_t n, const void* a, const void* b, double* out, void* stream) {
  return guard([&] {
    cudaStream_t s = S(stream);
    if (!t_scal.p) t_scal.alloc(1);
    if (n <= 0) {
      *out = 0.0;
      return;
    }
    if (dtype == 0)
      sg::launch_reduce<1>(n, DotT<double>{(const double*)a, (const double*)b},
                           sg::StoreTo<1>{{t_scal.p}}, t_red, s);
    else
      sg::launch_reduce<1>(n, DotT<float>{(const float*)a, (const float*)b},
                           sg::StoreTo<1>{{t_scal.p}}, t_red, s);
    SG_CUDA(cudaMemcpyAsync(out, t_scal.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
  });
}
int sg_vec_axpy(int dtype, int64_t n, double alpha, const void* x, void* y, void* stream) {
  return vec_op(dtype, 0, n, x, nullptr, y, alpha, stream);
}
int sg_vec_xpby(int dtype, int64_t n, const void* x, double beta, void* y, void* stream) {
  return vec_op(dtype, 1, n, x, nullptr, y, beta, stream);
}
int sg_vec_sub(int dtype, int64_t n, const void* a, const void* b, void* c, void* stream) {
  return vec_op(dtype, 2, n, a, b, c, 0.0, stream);
}
int sg_vec_mul(int dtype, int64_t n, const void* a, const void* b, void* c, void* stream) {
  return vec_op(dtype, 3, n, a, b, c, 0.0, stream);
}
int sg_vec_scale(int dtype, int64_t n, const void* a, double s, void* c, void* stream) {
  return vec_op(dtype, 4, n, a, nullptr, c, s, stream);
}
int sg_vec_div(int dtype, int64_t n, const void* a, double s, void* c, void* stream) {
  return vec_op(dtype, 5, n, a, nullptr, c, s, stream);
}
int sg_vec_bf16(int64_t n, const float* a, float* b, void* stream) {
  return guard([&] {
    if (n <= 0) return;
    bf16_kernel<<<sg::grid_blocks(n, 256), 256, 0, S(stream)>>>(n, a, b);
    SG_CHECK_LAUNCH();
  });
}

int sg_make_state(int kind, int nx, int ny, int nz, double vf, double floor_, uint64_t seed,
                  double* rho, void* stream) {
  return guard([&] {
    SG_REQUIRE(kind >= 0 && kind <= 5, "unknown state kind");
    SG_REQUIRE(nx > 0 && ny > 0 && nz > 0 && rho, "bad fixture arguments");
    sg::make_state_device(kind, nx, ny, nz, vf, floor_, static_cast<unsigned long long>(seed), rho,
                          S(stream));
  });
}

}  // extern "C"

// ------------------------------------------------- standalone transfers
struct sg_transfer {
  sg::Grid fine, coarse;
};

extern "C" {

int sg_transfer_create(int nx, int ny, int nz, const uint8_t* mask, sg_transfer** out) {
  return guard([&] {
    auto t = std::make_unique<sg_transfer>();
    sg::build_grid(t->fine, nx, ny, nz, mask, 0);
    sg::build_coarse_grid(t->fine, t->coarse, 0);
    *out = t.release();
  });
}

void sg_transfer_destroy(sg_transfer* t) { delete t; }

int sg_transfer_coarse_mask(sg_transfer* t, uint8_t* mask) {
  return guard([&] {
    const int64_t nn = t->coarse.d.nnodes();
    for (int64_t n = 0; n < nn; ++n)
      for (int a = 0; a < 3; ++a) mask[3 * n + a] = (t->coarse.h_nmask[size_t(n)] >> a) & 1;
  });
}

int sg_transfer_apply(sg_transfer* t, int transpose, const double* x, double* y, void* stream) {
  return guard([&] {
    cudaStream_t s = S(stream);
    sg::DBuf<double> a(static_cast<size_t>(3 * t->fine.d.nnodes())),
        c(static_cast<size_t>(3 * t->coarse.d.nnodes()));
    if (transpose) {
      sg::scatter_free<double>(t->fine, x, a.p, s);
      sg::restrict_(t->fine, t->coarse, a.p, c.p, s);
      sg::gather_free<double>(t->coarse, c.p, y, s);
    } else {
      sg::scatter_free<double>(t->coarse, x, c.p, s);
      sg::prolong(t->fine, t->coarse, c.p, a.p, false, s);
      sg::gather_free<double>(t->fine, a.p, y, s);
    }
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

int sg_transfer_csr(sg_transfer* t, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) {
  return guard([&] { sg::transfer_export_csr(t->fine, t->coarse, indptr, indices, data, nnz, 0); });
}

int sg_level1_csr(sg_fine* f, const double* triples, const uint32_t* codes, const double* diffs,
                  int ncodes, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(f->mu);
    sg::Grid coarse;
    sg::build_coarse_grid(f->op.grid, coarse, 0);
    sg::L1Tables tb;
    std::memcpy(tb.tri, triples, sizeof(double) * 8 * 576);
    tb.codes.assign(codes, codes + ncodes);
    tb.diffs.assign(diffs, diffs + size_t(ncodes) * 576);
    sg::DBuf<double> A(static_cast<size_t>(243 * coarse.d.nnodes()));
    sg::galerkin_level1(f->op, coarse, tb, A.p, 0);
    const int64_t n = sg::stencil_count_nnz(coarse, A.p, 0);
    *nnz = n;
    if (indices) sg::stencil_export_csr(coarse, A.p, indptr, indices, data, 0);
  });
}

}  // extern "C"

namespace sg {
unsigned long long g_sg_launches = 0;
}

extern "C" {

uint64_t sg_launch_count(void) { return __atomic_load_n(&sg::g_sg_launches, __ATOMIC_RELAXED); }

int sg_fine_apply_nodes(sg_fine* f, int tag, const void* u, void* y, void* stream) {
  return guard([&] { sg::fine_apply_tag(f->op, tag, u, y, S(stream)); });
}

int64_t sg_fine_n_nodes(const sg_fine* f) { return f ? f->op.grid.d.nnodes() : -1; }

}  // extern "C"

// Per-kernel device timings for bench.py (CUDA events on the launch stream,
// L2 flushed by a 256 MiB memset before every timed repetition).
extern "C" int sg_hier_profile(sg_hier* h, int what, int reps, double* ms_avg, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    sg::Hier& H = *h->h;
    sg::Level& L0 = *H.lv[0];
    const int64_t nd0 = L0.nd();
    sg::DBuf<double> a(static_cast<size_t>(nd0)), b(static_cast<size_t>(nd0));
    sg::DBuf<float> fa(static_cast<size_t>(nd0)), fb(static_cast<size_t>(nd0));
    const size_t n32 = size_t(sg::p32_size(H.fine->grid.d));
    sg::DBuf<float> pa(n32), pb(n32);
    pa.zero(s);
    sg::DBuf<uint8_t> flush(size_t(256) << 20);
    // inputs: seeded unit gaussian vectors (free DOFs; fixed entries 0), not zeros
    sg::fill_gaussian_unit(*L0.g, 12345u, a.p, H.red, H.scal.p + 3, s);
    sg::cvt_f64_to_f32(nd0, a.p, fa.p, s);
    if (sg::p32_supported(*H.fine)) sg::to_p32<double>(H.fine->grid.d, a.p, pa.p, s);
    for (size_t l = 1; l < H.lv.size(); ++l)
      sg::fill_gaussian_unit(*H.lv[l]->g, 777u + l, H.lv[l]->w.r.p, H.red, H.scal.p + 3, s);
    cudaEvent_t e0, e1;
    SG_CUDA(cudaEventCreate(&e0));
    SG_CUDA(cudaEventCreate(&e1));
    double total = 0.0;
    for (int r = 0; r < reps; ++r) {
      SG_CUDA(cudaMemsetAsync(flush.p, r & 0xff, flush.n, s));
      // 8 / 9: the coarsest solve right after another coarsest solve / after the
      // restriction onto the coarsest level (launch-transition cost probes)
      if (what == 8) sg::coarsest_solve(H, H.lv.back()->w.r.p, H.lv.back()->w.x.p, s);
      if (what == 9 && H.lv.size() > 1)
        sg::restrict_(*H.lv[H.lv.size() - 2]->g, *H.lv.back()->g, H.lv[H.lv.size() - 2]->w.r.p,
                      H.lv.back()->w.r.p, s);
      SG_CUDA(cudaEventRecord(e0, s));
      switch (what) {
        case 0:  // the level-0 FP32 apply the V-cycle runs (P32 layout when supported)
          if (sg::p32_supported(*H.fine)) sg::fine_apply_p32(*H.fine, pa.p, pb.p, s);
          else sg::fine_apply_f32(*H.fine, fa.p, fb.p, s);
          break;
        case 1: sg::fine_apply_f64(*H.fine, a.p, b.p, s); break;
        case 2: {
          SG_REQUIRE(H.lv.size() > 1, "no level 1");
          sg::Level& L1 = *H.lv[1];
          if (L1.st.T64s.p)  // the symmetric copy the single-GPU cycle reads
            sg::stencil_sym64(*L1.g, L1.st.T64s.p, 0, L1.w.r.p, L1.w.y64.p, nullptr, nullptr, nullptr, 0.0,
                              0.0, true, s);
          else
            sg::stencil_apply<double>(*L1.g, L1.st.T64.p, L1.w.r.p, L1.w.y64.p, s);
          break;
        }
        case 3:
        case 8:
        case 9: {
          sg::Level& Lc = *H.lv.back();
          sg::coarsest_solve(H, Lc.w.r.p, Lc.w.x.p, s);
          break;
        }
        case 4: sg::cycle_run(H, 1, s); break;
        case 5: sg::fine_apply_bf16(*H.fine, fa.p, fb.p, s); break;
        case 6: {  // the fused level-0 apply + Chebyshev step the V-cycle runs (P32)
          SG_REQUIRE(H.lv[0]->p32, "level 0 is not in the P32 layout");
          sg::Level& L = *H.lv[0];
          sg::fine_apply_p32_cheb(*H.fine, L.w.x32.p, L.w.x32b.p, L.w.b32.p, L.dinv32p.p, L.w.dd32.p,
                                  0.5f, 0.25f, false, s);
          break;
        }
        case 7: {  // the fused level-0 apply + residual the V-cycle runs (P32 -> node f64)
          SG_REQUIRE(H.lv[0]->p32, "level 0 is not in the P32 layout");
          sg::Level& L = *H.lv[0];
          sg::fine_apply_p32_res(*H.fine, pa.p, a.p, b.p, s);
          (void)L;
          break;
        }
        default: throw sg::Error("unknown profile target");
      }
      SG_CUDA(cudaEventRecord(e1, s));
      SG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      SG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_avg = total / std::max(reps, 1);
  });
}

// Development instrumentation: %globaltimer stamps (ns) of every pcg80 block at
// its phase boundaries; pipelined brick kernel: steps 8..15, 8 stamps each.
// out: 64 * 256 int64.
extern "C" int sg_hier_pcg80_trace(sg_hier* h, long long* out, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = S(stream);
    sg::Hier& H = *h->h;
    SG_REQUIRE(H.coarsest_mode == 1, "coarsest solver is not pcg80");
    sg::DBuf<long long> t(64 * 256);
    t.zero(s);
    sg::Level& Lc = *H.lv.back();
    H.pcg.trace = t.p;
    sg::coarsest_solve(H, Lc.w.r.p, Lc.w.x.p, s);
    H.pcg.trace = nullptr;
    t.download(out, 64 * 256, s);
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

namespace sg {
void* ptap_compute(int64_t nf, int64_t nc, const int64_t* Pp, const int64_t* Pj, const double* Px,
                   const int64_t* Kp, const int64_t* Kj, const double* Kx, int64_t* nnz,
                   cudaStream_t s);
void ptap_fetch(void* h, int64_t* Cp, int64_t* Cj, double* Cx);
void ptap_free(void* h);
}  // namespace sg

extern "C" {

int sg_ptap_csr(int64_t nf, int64_t nc, const int64_t* Pp, const int64_t* Pj, const double* Px,
                const int64_t* Kp, const int64_t* Kj, const double* Kx, void** result,
                int64_t* nnz, void* stream) {
  return guard([&] {
    *result = sg::ptap_compute(nf, nc, Pp, Pj, Px, Kp, Kj, Kx, nnz, S(stream));
  });
}

int sg_csr_result_get(void* result, int64_t* Cp, int64_t* Cj, double* Cx) {
  return guard([&] { sg::ptap_fetch(result, Cp, Cj, Cx); });
}

void sg_csr_result_free(void* result) { sg::ptap_free(result); }

}  // extern "C"

// Host-only work plans (no device needed): the pcg80 brick split and the P32
// fine-apply tiling, exposed so their partition invariants are tested on CPU.
extern "C" int sg_plan_brick(int nx, int ny, int nz, int nsm, int32_t* out3) {
  return guard([&] {
    sg::GridDesc g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    int sx = 0, sy = 0, sz = 0;
    const bool ok = sg::brick_plan(g, nsm, sx, sy, sz);
    out3[0] = ok ? sx : 0;
    out3[1] = ok ? sy : 0;
    out3[2] = ok ? sz : 0;
  });
}
extern "C" int sg_plan_p32_bs(int nx, int ny, int nz, int nsm, int nt, int32_t* out7) {
  return guard([&] {
    SG_REQUIRE(nt == 256 || nt == 512, "sg_plan_p32_bs: block size 256 or 512");
    sg::GridDesc g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    const sg::PkPlan pl = sg::pk_plan(g, nsm, nt);
    const int v[7] = {pl.P, pl.T, pl.SX, pl.R, pl.tilesy, pl.kchunk, pl.nch};
    for (int i = 0; i < 7; ++i) out7[i] = v[i];
  });
}
extern "C" int sg_plan_p32(int nx, int ny, int nz, int nsm, int32_t* out7) {
  sg::GridDesc g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  return sg_plan_p32_bs(nx, ny, nz, nsm, sg::pk_threads(g, 0), out7);
}
