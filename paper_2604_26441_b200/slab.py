"""Multi-GPU slab partition of the PCG / GMG solve.

The reference is single-process (``krylov.pcg``, krylov.py:113-165, called as
``pcg(op.matvec, h.vcycle, b, cfg)`` by bench/runner.py:66-88); BASELINE.json's
north star asks for the fine and first coarse levels to be slab-partitioned
over the GPUs of one node with halo exchange and a dot-product allreduce, and
the deeper levels gathered.  This module is that layer:

* ``slab_plan`` -- z-slab ownership per level.  The partition is made on the
  coarsest slab level (node planes split as evenly as possible) and inherited
  by the finer one (coarse plane c <-> fine plane 2c), so the window of every
  rank is a self-consistent sub-grid: fine window = the fine image of the
  coarse window, starting on an even plane.  Ghost planes: the level-0 window
  carries the two fine planes below its first owned plane and one above; the
  level-1 window one plane on each side.  Every operator input is halo-filled
  first, so owned rows are computed from exactly the single-GPU operands.
* ``TorchSlabComm`` -- the three data movements (ghost-plane exchange, rank
  ordered sum of a few doubles, allgather of owned planes) on torch tensors
  over ``torch.distributed``: NCCL on CUDA tensors, or gloo (host staged).
* ``SlabSolver`` -- one rank's handle: builds its windows in libsg_b200.so
  from the replicated hierarchy and runs the native PCG / FGMRES drivers over
  them (``sg_dist_solve``).  Two transports:
    - ``"peer"`` (default with NCCL): the exchanges are device kernels that
      store into the other ranks' mailboxes (CUDA IPC mappings over NVLink,
      ``sg_dist_create_peer``, csrc/sg_peer.cu) and signal with system-scope
      flags -- no host step inside a solve iteration except the one scalar
      read of the PCG driver, and the distributed cycle replays from a CUDA
      graph.
    - ``"torch"``: the library calls back into ``TorchSlabComm`` for each
      exchange (gloo / NCCL through torch.distributed).
  Every rank passes the same global ``b`` and receives the same global ``x``.

Levels below the slab levels are replicated on every rank: the cut level's
residual is allgathered, each rank runs the coarse tail, and slices its own
window out of the prolonged correction (no broadcast step).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = ["slab_plan", "halo_pieces", "TorchSlabComm", "SlabSolver", "slab_pcg"]


@dataclass(frozen=True)
class Window:
    w0: int  # first window node plane (global, this level)
    w1: int  # last window node plane (inclusive)
    o0: int  # first owned node plane
    o1: int  # one past the last owned node plane

    @property
    def n_planes(self) -> int:
        return self.w1 - self.w0 + 1


def _split(n: int, world: int):
    q, rem = divmod(n, world)
    out, a = [], 0
    for r in range(world):
        b = a + q + (1 if r < rem else 0)
        out.append((a, b))
        a = b
    return out


def slab_plan(nz: int, world: int, n_dist: int):
    """plan[level][rank] -> Window for a fine grid of ``nz`` element layers.

    n_dist = 1: only level 0 is partitioned (1 ghost plane each side).
    n_dist = 2: levels 0 and 1 (requires even nz); ownership is split on the
    nz/2 + 1 coarse node planes.
    """
    if n_dist not in (1, 2):
        raise ValueError("n_dist must be 1 or 2")
    if world < 1:
        raise ValueError("world must be >= 1")
    if n_dist == 1:
        if world > nz + 1:
            raise ValueError(f"{world} ranks but only {nz + 1} node planes")
        lv0 = []
        for a, b in _split(nz + 1, world):
            lv0.append(Window(max(a - 1, 0), min(b, nz), a, b))
        return [lv0]
    if nz % 2:
        raise ValueError("two slab levels need an even number of element layers")
    nzc = nz // 2
    if world > nzc + 1:
        raise ValueError(f"{world} ranks but only {nzc + 1} coarse node planes")
    lv0, lv1 = [], []
    for c0, c1 in _split(nzc + 1, world):
        w1 = Window(max(c0 - 1, 0), min(c1, nzc), c0, c1)
        lv1.append(w1)
        lv0.append(Window(2 * w1.w0, min(2 * w1.w1, nz), 2 * c0, min(2 * c1, nz + 1)))
    return [lv0, lv1]


def _owner(plan_level, p):
    for r, w in enumerate(plan_level):
        if w.o0 <= p < w.o1:
            return r
    raise ValueError(f"plane {p} has no owner")


def halo_pieces(plan_level):
    """Canonical list of ghost transfers of one level: (src, dst, p0, p1),
    planes [p0, p1) owned by src and ghost on dst, in (dst, plane) order --
    the order both sides of every pair enumerate their sends / receives."""
    out = []
    for dst, w in enumerate(plan_level):
        for lo, hi in ((w.w0, w.o0), (w.o1, w.w1 + 1)):
            p = lo
            while p < hi:
                src = _owner(plan_level, p)
                q = min(hi, plan_level[src].o1)
                if src == dst:
                    raise ValueError("ghost plane owned by its own rank")
                out.append((src, dst, p, q))
                p = q
    return out


#: exchange level of level-0 vectors in the P32 layout (csrc/sg_hier.cuh kP32Level)
P32_LEVEL = 2


def p32_xs(nx: int) -> int:
    """Row stride of the P32 layout (csrc/sg_fine_pk.cu p32_xs): NX = nx + 1
    rounded up to a multiple of 32 up to 256, else to even."""
    nx1 = nx + 1
    return (nx1 + 31) & ~31 if nx1 <= 256 else (nx1 + 1) & ~1


class TorchSlabComm:
    """Slab data movement on torch tensors over a torch.distributed group.

    plane_sizes[l]: values per node plane on level l (3 (nx+1)(ny+1)).
    full_planes[l]: node planes of the whole level-l grid.
    """

    def __init__(self, plan, plane_sizes, full_planes, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if len(plan[0]) != self.world:
            raise ValueError("plan was made for a different world size")
        self.plan = plan
        self.psz = list(plane_sizes)
        self.full_planes = list(full_planes)
        self.backend = dist.get_backend(group)
        self.nccl = self.backend == "nccl"
        self.pieces = [halo_pieces(lv) if lv is not None else [] for lv in plan]
        self.n_halo = 0
        self.n_gather = 0
        self.n_sum = 0

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _stage(self, t):
        return t if self.nccl or not t.is_cuda else t.cpu()

    # -- ghost planes -----------------------------------------------------
    def halo(self, level: int, vec):
        """Fill the ghost planes of this rank's window vector of ``level``."""
        w = self.plan[level][self.rank]
        ps = self.psz[level]
        if vec.numel() != w.n_planes * ps:
            raise ValueError("window vector size does not match the plan")
        self.n_halo += 1
        ops, post = [], []
        for tag, (src, dst, p0, p1) in enumerate(self.pieces[level]):
            if src == self.rank:
                buf = vec[(p0 - w.w0) * ps:(p1 - w.w0) * ps]
                ops.append(("send", self._stage(buf), dst, tag))
            elif dst == self.rank:
                view = vec[(p0 - w.w0) * ps:(p1 - w.w0) * ps]
                buf = view if self.nccl or not view.is_cuda else view.new_empty(view.shape, device="cpu")
                ops.append(("recv", buf, src, tag))
                if buf is not view:
                    post.append((view, buf))
        if not ops:
            return
        d = self.dist
        if self.nccl:
            p2p = [d.P2POp(d.isend if k == "send" else d.irecv, t, self._peer(peer), self.group)
                   for k, t, peer, _ in ops]
            for req in d.batch_isend_irecv(p2p):
                req.wait()
        else:
            reqs = [(d.isend if k == "send" else d.irecv)(t, self._peer(peer), self.group, tag)
                    for k, t, peer, tag in ops]
            for req in reqs:
                req.wait()
        for view, buf in post:
            view.copy_(buf)

    # -- rank-ordered sum -------------------------------------------------
    def allreduce(self, vals):
        """vals (n doubles) <- sum over ranks, accumulated in rank order."""
        self.n_sum += 1
        if self.world == 1:
            return
        src = self._stage(vals.contiguous())
        parts = [src.new_empty(src.shape) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        vals.copy_(acc)

    # -- owned planes -> full vector ---------------------------------------
    def allgather(self, level: int, win, full):
        self.n_gather += 1
        lv = self.plan[level]
        ps = self.psz[level]
        w = lv[self.rank]
        if full.numel() != self.full_planes[level] * ps:
            raise ValueError("full vector size does not match the level")
        own = win[(w.o0 - w.w0) * ps:(w.o1 - w.w0) * ps]
        if self.world == 1:
            full[w.o0 * ps:w.o1 * ps].copy_(own)
            return
        nmax = max(x.o1 - x.o0 for x in lv) * ps
        src = self._stage(own.new_zeros(nmax))
        src[:own.numel()].copy_(own)
        parts = [src.new_empty(nmax) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        for r, x in enumerate(lv):
            n = (x.o1 - x.o0) * ps
            full[x.o0 * ps:x.o1 * ps].copy_(parts[r][:n])


# ------------------------------------------------------------ ctypes glue
class _DevArray:
    """Zero-copy torch view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _wrap(ptr, n, elem_bytes):
    import torch
    typestr = "<f8" if elem_bytes == 8 else "<f4"
    return torch.as_tensor(_DevArray(ptr, n, typestr), device="cuda")


def _guarded(fn):
    def call(*args):
        try:
            fn(*args)
            return 0
        except Exception as exc:  # a raising ctypes callback would report success
            import sys
            print(f"slab comm callback failed: {exc!r}", file=sys.stderr)
            return 1
    return call


class _TorchRank:
    def __init__(self, group):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def barrier(self):
        self.dist.barrier(self.group)

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class SlabSolver:
    """This rank's part of a slab-partitioned solve of ``op`` preconditioned by
    ``hierarchy`` (built identically on every rank).

    ``n_dist`` slab levels (default: 2 when the hierarchy has >= 3 levels and
    even nz, else 1); the rest of the hierarchy is the replicated coarse tail.
    ``transport``: "peer" (device kernels over IPC-mapped mailboxes), "torch"
    (host callbacks into TorchSlabComm) or "auto" (peer with NCCL, torch
    otherwise).  ``group``: a torch.distributed group (None = WORLD).  One
    process per GPU: a peer wait kernel spins on the device, so ranks sharing
    a CUDA context (threads) could deadlock on an implicitly synchronising
    runtime call (cudaFree) in another rank.
    ``release_full``: free the hierarchy's replicated full-grid copies of the
    slab levels once the windows exist (the hierarchy's own single-GPU cycle
    is then unavailable); only the windows and the coarse tail stay resident.
    """

    def __init__(self, op, hierarchy, group=None, n_dist=None, transport="auto",
                 release_full=False):
        from . import _dev
        if hierarchy._op is not op:
            raise ValueError("hierarchy built for a different operator")
        nl = hierarchy.n_levels
        if nl < 2:
            raise ValueError("slab partition needs at least two hierarchy levels")
        g = op.grid
        if n_dist is None:
            n_dist = 2 if (nl >= 3 and g.nz % 2 == 0) else 1
        if n_dist >= nl:
            raise ValueError("need a replicated level below the slab levels")
        grp = _TorchRank(group)
        world, rank = grp.world, grp.rank
        if transport == "auto":
            transport = "peer" if grp.dist.get_backend(group) == "nccl" else "torch"
        if transport not in ("peer", "torch"):
            raise ValueError(f"unknown slab transport {transport!r}")
        self.transport = transport
        self._grp = grp
        self.plan = slab_plan(g.nz, world, n_dist)
        dims = [hierarchy.levels[l]._dims for l in range(n_dist)]
        psz = [3 * (nx + 1) * (ny + 1) for nx, ny, _ in dims]
        fpl = [nz + 1 for _, _, nz in dims]
        # exchange level 2 (P32_LEVEL): level 0 in the P32 layout of the FP32
        # level-0 smoother -- the same planes, 3 * XS * (ny + 1) floats each
        while len(psz) < P32_LEVEL:
            psz.append(0)
            fpl.append(0)
        psz.append(3 * p32_xs(g.nx) * (g.ny + 1))
        fpl.append(g.nz + 1)
        plan_x = list(self.plan) + [None] * (P32_LEVEL - n_dist) + [self.plan[0]]
        self.comm = TorchSlabComm(plan_x, psz, fpl, group) if transport == "torch" else None
        self.op, self.hierarchy, self.n_dist = op, hierarchy, n_dist
        self._psz = psz
        mine = [self.plan[l][rank] for l in range(n_dist)]
        mine_x = mine + [None] * (P32_LEVEL - n_dist) + [mine[0]]
        self._nwin = [w.n_planes * p if w else 0 for w, p in zip(mine_x, psz)]
        self._nfull = [f * p for f, p in zip(fpl, psz)]
        self._lib = _native.load()
        if transport == "peer":
            self._init_peer(hierarchy, n_dist, rank, world, release_full)
            return
        c = self.comm

        def halo(_ctx, level, vec, eb, _stream):
            c.halo(level, _wrap(vec, self._nwin[level], eb))

        def allreduce(_ctx, vals, n, _stream):
            c.allreduce(_wrap(vals, n, 8))

        def allgather(_ctx, level, win, full, _stream):
            c.allgather(level, _wrap(win, self._nwin[level], 8), _wrap(full, self._nfull[level], 8))

        # keep the CFUNCTYPE objects alive as long as the native handle
        self._cbs = _native.Comm(None, _native.HALO_FN(_guarded(halo)),
                                _native.ALLREDUCE_FN(_guarded(allreduce)),
                                _native.ALLGATHER_FN(_guarded(allgather)))
        planes = np.array([[w.w0, w.w1, w.o0, w.o1] for w in mine], dtype=np.int32)
        h = ctypes.c_void_p()
        grp.barrier()  # first collective of the group before any P2P
        _native.check(self._lib.sg_dist_create(hierarchy._hh, n_dist, planes.ctypes.data,
                                               ctypes.byref(self._cbs), _dev.stream(),
                                               ctypes.byref(h)))
        self._hd = h
        if release_full:
            _native.check(self._lib.sg_dist_release_full(self._hd, _dev.stream()))

    def _init_peer(self, hierarchy, n_dist, rank, world, release_full):
        """Device transport: create the mailbox, exchange its CUDA IPC handle
        over the process group and map every peer's."""
        from . import _dev
        planes = np.array([[[w.w0, w.w1, w.o0, w.o1] for w in (self.plan[l][r] for l in range(n_dist))]
                           for r in range(world)], dtype=np.int32)
        h = ctypes.c_void_p()
        _native.check(self._lib.sg_dist_create_peer(hierarchy._hh, n_dist, planes.ctypes.data, rank,
                                                    world, _dev.stream(), ctypes.byref(h)))
        self._hd = h
        handle = (ctypes.c_char * 64)()
        base = ctypes.c_uint64()
        _native.check(self._lib.sg_dist_peer_handle(h, handle, ctypes.byref(base)))
        hs = self._grp.all_gather_object(bytes(handle))
        _native.check(self._lib.sg_dist_peer_open(h, b"".join(hs), None))
        if release_full:
            _native.check(self._lib.sg_dist_release_full(h, _dev.stream()))
        self._grp.barrier()  # every mailbox mapped and zeroed before the first exchange

    def close(self):
        hd = getattr(self, "_hd", None)
        if hd is not None and hd.value:
            if getattr(self, "transport", "torch") == "peer":
                # no rank unmaps / frees its mailbox while another may still store into it
                import torch
                torch.cuda.current_stream().synchronize()
                self._grp.barrier()
            self._lib.sg_dist_destroy(hd)
            self._hd = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_free(self) -> int:
        return self.op.n_free

    def _apply(self, what, x, ktag=None, gamma=1):
        from . import _dev
        xd, host = _dev.as_device(x, np.float64, self.n_free)
        y = _dev.empty(self.n_free)
        k = self.op.precision.code if ktag is None else ktag
        _native.check(self._lib.sg_dist_apply(self._hd, what, k, gamma, _dev.ptr(xd), _dev.ptr(y),
                                              _dev.stream()))
        return _dev.back(y, host)

    def matvec(self, x):
        """K x over the slabs (same global vector on every rank)."""
        return self._apply(0, x)

    def vcycle(self, r):
        return self._apply(1, r, gamma=1)

    def wcycle(self, r):
        return self._apply(1, r, gamma=2)

    def solve(self, b, cfg, method="pcg", gamma=1):
        from . import _dev
        from .krylov import SolveReport, _KINDS
        bd, host = _dev.as_device(b, np.float64, self.n_free)
        x = _dev.empty(self.n_free)
        hist = np.zeros(cfg.maxiter + 1)
        c = _native.SolverCfg(cfg.tol, cfg.maxiter, cfg.restart)
        rep = _native.Report()
        m = {"pcg": 0, "fgmres": 1}[method]
        _native.check(self._lib.sg_dist_solve(self._hd, m, self.op.precision.code, gamma,
                                              _dev.ptr(bd), _dev.ptr(x), ctypes.byref(c),
                                              ctypes.byref(rep), hist.ctypes.data, _dev.stream()))
        it = int(rep.iterations)
        return SolveReport(bool(rep.converged), it, float(rep.final_true_residual),
                           _KINDS[int(rep.failure_kind)],
                           [float(v) for v in hist[:it]] if cfg.record_history else [],
                           float(rep.wall_time), _dev.back(x, host))

    def pcg(self, b, cfg):
        """pcg(op.matvec, h.vcycle, b, cfg) over the slabs (krylov.py:113-165)."""
        return self.solve(b, cfg, "pcg")

    def fgmres(self, b, cfg):
        """fgmres(op.matvec, h.vcycle, b, cfg) over the slabs (krylov.py:168-281)."""
        return self.solve(b, cfg, "fgmres")


def slab_pcg(op, hierarchy, b, cfg, group=None, transport="auto"):
    """One-shot slab-partitioned ``pcg(op.matvec, hierarchy.vcycle, b, cfg)``."""
    s = SlabSolver(op, hierarchy, group, transport=transport)
    try:
        return s.pcg(b, cfg)
    finally:
        s.close()
