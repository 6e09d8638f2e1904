"""Development aid: per-block pcg80 phase times (cycle stamps; build with
SG_NVCC_EXTRA=-DSG_TRACE_CLOCK) against the brick size -- is the step period
set by the largest bricks?"""
import os, sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
lib = _native.load()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
h.vcycle(np.ones(g.n_free))
t = np.zeros(64 * 256, dtype=np.int64)
_native.check(lib.sg_hier_pcg80_trace(h._hh, t.ctypes.data, _dev.stream()))
t = t.reshape(256, 8, 8)
nb = int((t[:, 0, 0] > 0).sum())
t = t[:nb].astype(np.float64) / 1.965e3
n = N // 4 + 1
sx, sy, sz = 3, 7, 7
sizes = []
for b in range(nb):
    bx, by, bz = b % sx, (b // sx) % sy, b // (sx * sy)
    d = lambda i, s: (i + 1) * n // s - i * n // s
    sizes.append(d(bx, sx) * d(by, sy) * d(bz, sz))
sizes = np.array(sizes)
ph = {"publish": (0, 1), "fill": (1, 5), "spmv": (5, 3), "validate": (3, 6), "collect": (6, 2), "update": (2, 4)}
for name, (a, b) in ph.items():
    v = np.median(t[:, :, b] - t[:, :, a], axis=1)
    print(f"{name:9s}", " ".join(f"{s}:{v[sizes == s].mean():.3f}" for s in sorted(set(sizes))))
