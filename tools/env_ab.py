"""Development aid: one environment switch swept over values -- V-cycle
bit-identity against the first value, sg_hier_profile times (level-1 SpMV,
V-cycle).  python tools/env_ab.py VAR v0,v1,... [N ...]"""
import os, subprocess, sys
import numpy as np
code = r'''
import ctypes, sys, warnings, numpy as np; sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[2])
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("random_floor", N, N, N, vf=0.5, seed=42), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
r = P.SplitMix64(7).gaussian(g.n_free)
np.save(sys.argv[1], h.vcycle(r))
lib = _native.load()
res = []
for what in (2, 4):
    out = ctypes.c_double()
    _native.check(lib.sg_hier_profile(h._hh, what, 30, ctypes.byref(out), _dev.stream()))
    res.append(out.value * 1e3)
print("l1 spmv %.2f us  vcycle %.1f us" % tuple(res))
'''
var, vals = sys.argv[1], sys.argv[2].split(",")
for N in (sys.argv[3:] or ["100", "200"]):
    base = None
    for v in vals:
        path = f"/tmp/envab_{v}.npy"
        p = subprocess.run([sys.executable, "-c", code, path, N], env=dict(os.environ, **{var: v}),
                           capture_output=True, text=True)
        if p.returncode:
            print(N, v, "FAILED", p.stderr[-600:]); continue
        x = np.load(path)
        base = x if base is None else base
        print(f"N={N} {var}={v:4s} {p.stdout.strip()}  identical={bool(np.array_equal(x, base))}", flush=True)
