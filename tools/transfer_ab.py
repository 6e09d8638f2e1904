"""Development aid: structured transfers, pair/row kernels vs the per-node
kernels (SG_PROLONG_NODE / SG_RESTRICT_NODE): V-cycle bit-identity and time."""
import os, subprocess, sys
import numpy as np
code = r'''
import ctypes, sys, warnings, numpy as np; sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
dims = tuple(int(v) for v in sys.argv[2].split(","))
g = P.build_cantilever(*dims)
kind = sys.argv[4]
op = P.FineOperator(g, P.simp_modulus(P.make_state(kind, *dims, vf=0.5, seed=42), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, sys.argv[3])
r = P.SplitMix64(7).gaussian(g.n_free)
np.save(sys.argv[1], h.vcycle(r))
lib = _native.load()
out = ctypes.c_double()
_native.check(lib.sg_hier_profile(h._hh, 4, 30, ctypes.byref(out), _dev.stream()))
print("vcycle %.1f us" % (out.value * 1e3))
'''
cases = [a.split(":") for a in (sys.argv[1:] or ["100,100,100:fp32:uniform", "64,48,40:fp32:random_floor",
                                                  "64,48,40:fp64:random_floor", "33,17,9:fp64:binary",
                                                  "200,200,200:fp32:uniform"])]
for dims, pol, kind in cases:
    res = {}
    for name, env in (("new", {}), ("old", {"SG_PROLONG_NODE": "1", "SG_RESTRICT_NODE": "1"})):
        path = f"/tmp/tr_{name}.npy"
        p = subprocess.run([sys.executable, "-c", code, path, dims, pol, kind],
                           env=dict(os.environ, **env), capture_output=True, text=True)
        if p.returncode:
            print(dims, name, "FAILED", p.stderr[-800:]); break
        res[name] = (np.load(path), p.stdout.strip())
    if len(res) == 2:
        print(dims, pol, kind, "identical=%s" % np.array_equal(res["new"][0], res["old"][0]),
              "new:", res["new"][1], "old:", res["old"][1], flush=True)
