"""Development aid: FP64 apply under an environment switch -- output bit-identity
against the first value and sg_hier_profile time.  python tools/p64_ab.py VAR v0,v1 [N ...]"""
import os, subprocess, sys
import numpy as np
code = r'''
import ctypes, sys, warnings, numpy as np; sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
dims = tuple(int(v) for v in sys.argv[2].split(","))
g = P.build_cantilever(*dims)
op = P.FineOperator(g, P.simp_modulus(P.make_state("random_floor", *dims, vf=0.5, seed=42), 3.0))
u = P.SplitMix64(3).gaussian(g.n_free)
np.save(sys.argv[1], op.matvec(u))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
out = ctypes.c_double()
_native.check(_native.load().sg_hier_profile(h._hh, 1, 30, ctypes.byref(out), _dev.stream()))
print("fp64 apply %.2f us" % (out.value * 1e3))
'''
var, vals = sys.argv[1], sys.argv[2].split(",")
for dims in (sys.argv[3:] or ["100,100,100", "64,48,40", "200,200,200"]):
    base = None
    for v in vals:
        env = dict(os.environ)
        if v != "-":
            env[var] = v
        p = subprocess.run([sys.executable, "-c", code, "/tmp/p64ab.npy", dims], env=env,
                           capture_output=True, text=True)
        if p.returncode:
            print(dims, v, "FAILED", p.stderr[-600:]); continue
        x = np.load("/tmp/p64ab.npy")
        base = x if base is None else base
        print(f"{dims} {var}={v:3s} {p.stdout.strip()}  identical={bool(np.array_equal(x, base))}", flush=True)
