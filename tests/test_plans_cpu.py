"""CPU checks of the host-side work plans of the two hot kernels (C ABI, no
device): the pcg80 brick split partitions the coarsest node grid into at most
one brick per SM, and the P32 fine-apply tiling gives every node exactly one
owner in x, y and z (the ownership rules of csrc/sg_fine_pk.cu restated)."""

import ctypes

import numpy as np
import pytest

from paper_2604_26441_b200 import _native

KBR_CAP, KBR_WIN = 144, 448


def _brick(n, nsm=148):
    out = (ctypes.c_int32 * 3)()
    _native.check(_native.load().sg_plan_brick(n[0], n[1], n[2], nsm, out))
    return tuple(out)


def _p32(n, nsm=148, nt=None):
    out = (ctypes.c_int32 * 7)()
    if nt is None:
        _native.check(_native.load().sg_plan_p32(n[0], n[1], n[2], nsm, out))
    else:
        _native.check(_native.load().sg_plan_p32_bs(n[0], n[1], n[2], nsm, nt, out))
    return dict(zip(("P", "T", "SX", "R", "tilesy", "kchunk", "nch"), out))


@pytest.mark.parametrize("nodes", [(26, 26, 26), (16, 16, 16), (3, 2, 2), (7, 5, 4), (13, 26, 7)])
def test_brick_plan_partitions_the_coarsest_grid(nodes):
    NX, NY, NZ = nodes
    sx, sy, sz = _brick((NX - 1, NY - 1, NZ - 1))
    assert sx * sy * sz <= 148 and min(sx, sy, sz) >= 1
    owner = np.full((NZ, NY, NX), -1)
    for b in range(sx * sy * sz):   # balanced splits as in pcg80_brick_kernel
        bx, by, bz = b % sx, (b // sx) % sy, b // (sx * sy)
        x0, x1 = bx * NX // sx, (bx + 1) * NX // sx
        y0, y1 = by * NY // sy, (by + 1) * NY // sy
        z0, z1 = bz * NZ // sz, (bz + 1) * NZ // sz
        vol = (x1 - x0) * (y1 - y0) * (z1 - z0)
        assert 0 < vol <= KBR_CAP
        assert (x1 - x0 + 2) * (y1 - y0 + 2) * (z1 - z0 + 2) <= KBR_WIN
        assert (owner[z0:z1, y0:y1, x0:x1] == -1).all()
        owner[z0:z1, y0:y1, x0:x1] = b
    assert (owner >= 0).all()


def test_brick_plan_100cube_coarsest():
    # configs[3]: 25^3 coarsest elements -> 26^3 nodes on 147 bricks of <= 144 nodes (9x4x4)
    assert sorted(_brick((25, 25, 25))) == [3, 7, 7]


@pytest.mark.parametrize("dims", [(100, 100, 100), (200, 200, 200), (1, 1, 1), (9, 33, 17),
                                  (127, 4, 3), (131, 7, 5), (257, 2, 3), (40, 40, 40)])
@pytest.mark.parametrize("nt", [None, 512, 256])
def test_p32_tiling_owns_every_node_once(dims, nt):
    nx, ny, nz = dims
    pl = _p32(dims, nt=nt)
    P, T, SX, R = pl["P"], pl["T"], pl["SX"], pl["R"]
    assert P <= 64 and P * R <= (nt or 512) and R >= 2
    # x: pair p of tile t covers elements xo+2p, xo+2p+1 and owns nodes in [own_lo, own_hi)
    xown = np.zeros(nx + 1, int)
    for t in range(T):
        xo = t * SX
        lo = 0 if t == 0 else xo + 2
        hi = nx + 1 if t == T - 1 else xo + 2 * P - 2
        for p in range(P):
            ex = xo + 2 * p
            for node in (ex, ex + 1):
                if lo <= node < hi:
                    # node ex needs the left pair inside the tile unless it is node 0
                    assert node == ex + 1 or p > 0 or ex == 0
                    xown[node] += 1
        assert xo + 2 * P - 1 >= min(hi, nx + 1) - 1
    assert (xown == 1).all()
    # y: tile t covers element rows t*(R-1)-1 ... +R-1, owns node rows ej+1 of local rows 0..R-2
    yown = np.zeros(ny + 1, int)
    for t in range(pl["tilesy"]):
        for r in range(R - 1):
            on = t * (R - 1) - 1 + r + 1
            if 0 <= on <= ny:
                yown[on] += 1
    assert (yown == 1).all()
    # z: chunk c owns node planes [c*kchunk, min((c+1)*kchunk, nz+1))
    zown = np.zeros(nz + 1, int)
    for c in range(pl["nch"]):
        zown[c * pl["kchunk"]:min((c + 1) * pl["kchunk"], nz + 1)] += 1
    assert (zown == 1).all()


def test_native_halo_pieces_match_python():
    """sg_plan_halo (the device transport's transfer lists, csrc/sg_peer.cu) and
    slab.py halo_pieces (the torch transport's) enumerate the same ghost pieces."""
    import ctypes
    import numpy as np
    from paper_2604_26441_b200 import _native
    from paper_2604_26441_b200.slab import halo_pieces, slab_plan
    lib = _native.load()
    for nz in (4, 6, 8, 12, 20, 50, 100):
        for world in range(1, 9):
            for n_dist in (1, 2):
                try:
                    plan = slab_plan(nz, world, n_dist)
                except ValueError:
                    continue
                for lv in plan:
                    w = np.array([[x.w0, x.w1, x.o0, x.o1] for x in lv], dtype=np.int32)
                    out = np.zeros(4 * 64 + 1, dtype=np.int32)
                    assert lib.sg_plan_halo(world, w.ctypes.data, out.ctypes.data, 64) == 0
                    n = int(np.argmax(out == -1)) // 4
                    got = [tuple(int(v) for v in out[4 * i:4 * i + 4]) for i in range(n)]
                    assert got == [tuple(p) for p in halo_pieces(lv)], (nz, world, n_dist)
