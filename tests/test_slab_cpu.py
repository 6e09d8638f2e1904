"""CPU tests of the multi-GPU slab partition (paper_2604_26441_b200/slab.py).

* the plan's windows contain every operand the owned rows need;
* the decomposition is exact: the CPU oracle's fine apply / transfers evaluated
  on every rank's window (ghost planes filled as the halo does) reproduce the
  global results bit for bit on the owned rows (oracle = checker only);
* TorchSlabComm over gloo with 2 and 3 processes: halo, rank-ordered sum and
  allgather move exactly the right planes.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2604_26441_b200.slab import halo_pieces, slab_plan

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("nz,world,n_dist", [(8, 2, 2), (8, 5, 2), (100, 8, 2), (200, 8, 2),
                                             (12, 3, 2), (7, 2, 1), (9, 10, 1), (100, 8, 1)])
def test_plan_invariants(nz, world, n_dist):
    plan = slab_plan(nz, world, n_dist)
    for lvl, lv in enumerate(plan):
        nzl = nz >> lvl
        owned = [p for w in lv for p in range(w.o0, w.o1)]
        assert owned == list(range(nzl + 1))  # a partition, in rank order
        for w in lv:
            assert 0 <= w.w0 <= w.o0 < w.o1 <= w.w1 + 1 <= nzl + 1
            # the operator stencil of every owned plane lies in the window
            assert w.w0 <= max(w.o0 - 1, 0) and min(w.o1, nzl) <= w.w1
        for src, dst, p0, p1 in halo_pieces(lv):
            assert abs(src - dst) == 1 and lv[src].o0 <= p0 < p1 <= lv[src].o1
    if n_dist == 2:
        for w0, w1 in zip(plan[0], plan[1]):
            assert w0.w0 == 2 * w1.w0 and w0.w1 == min(2 * w1.w1, nz)
            # restriction of owned coarse planes reads fine planes [2c0-1, 2c1-1]
            assert w0.w0 <= max(2 * w1.o0 - 1, 0) and min(2 * w1.o1 - 1, nz) <= w0.w1
            # prolongation of owned fine planes reads coarse planes [c0, c1]
            assert min(w1.o1, nz // 2) <= w1.w1
    with pytest.raises(ValueError):
        slab_plan(9, 2, 2)
    with pytest.raises(ValueError):
        slab_plan(4, 4, 2)


def _window_grid(O, g, w0, w1):
    plane = 3 * (g.nx + 1) * (g.ny + 1)
    return O.make_grid(g.nx, g.ny, w1 - w0, g.mask[w0 * plane:(w1 + 1) * plane])


@pytest.mark.parametrize("world", [2, 3])
def test_window_decomposition_is_exact(world):
    from oracle import simp_oracle as O
    nx, ny, nz = 6, 4, 10
    g, E, ke = O.problem(nx, ny, nz, kind="binary", p=3.0)
    gc = O.transfer(g)[1]
    P_glob = O.transfer(g)[0]
    rng = np.random.default_rng(3)
    u = rng.standard_normal(g.n_free)
    uc = rng.standard_normal(gc.n_free)
    full_u = np.zeros(g.n_dof)
    full_u[g.free] = u
    full_uc = np.zeros(gc.n_dof)
    full_uc[gc.free] = uc
    Ku = np.zeros(g.n_dof)
    Ku[g.free] = O.fine_apply(g, E, ke, u)
    Rf = np.zeros(gc.n_dof)
    Rf[gc.free] = P_glob.T @ u
    Pc = np.zeros(g.n_dof)
    Pc[g.free] = P_glob @ uc
    plan = slab_plan(nz, world, 2)
    pl0, pl1 = 3 * (nx + 1) * (ny + 1), 3 * (nx // 2 + 1) * (ny // 2 + 1)
    for r in range(world):
        w, wc = plan[0][r], plan[1][r]
        gw = _window_grid(O, g, w.w0, w.w1)
        Ew = E.reshape(nz, ny * nx)[w.w0:w.w1].ravel()
        uw_full = full_u[w.w0 * pl0:(w.w1 + 1) * pl0]
        y = np.zeros(gw.n_dof)
        y[gw.free] = O.fine_apply(gw, Ew, ke, uw_full[gw.free])
        own = slice((w.o0 - w.w0) * pl0, (w.o1 - w.w0) * pl0)
        assert np.array_equal(y[own], Ku[w.o0 * pl0:w.o1 * pl0])
        # transfers between the two windows
        Pw, gcw = O.transfer(gw)
        assert (gcw.nz, gcw.nx) == (wc.w1 - wc.w0, nx // 2)
        rc = np.zeros(gcw.n_dof)
        rc[gcw.free] = Pw.T @ uw_full[gw.free]
        ownc = slice((wc.o0 - wc.w0) * pl1, (wc.o1 - wc.w0) * pl1)
        assert np.array_equal(rc[ownc], Rf[wc.o0 * pl1:wc.o1 * pl1])
        ucw_full = full_uc[wc.w0 * pl1:(wc.w1 + 1) * pl1]
        pf = np.zeros(gw.n_dof)
        pf[gw.free] = Pw @ ucw_full[gcw.free]
        assert np.array_equal(pf[own], Pc[w.o0 * pl0:w.o1 * pl0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run_ranks(mode, world, out, timeout=600):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "slab_worker.py"), mode,
                                       str(out)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=timeout)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-4000:]
    return json.load(open(out))


@pytest.mark.parametrize("world", [2, 3])
def test_torch_slab_comm_gloo(world, tmp_path):
    res = run_ranks("comm", world, tmp_path / "comm.json", timeout=300)
    assert len(res) == world
    for r in res:
        for k, v in r.items():
            assert (all(v) if isinstance(v, list) else v), (k, v)
