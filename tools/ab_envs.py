"""Development aid: V-cycle outputs under kernel-path switches (bit-identity A/B)."""
import os, subprocess, sys
import numpy as np
code = r'''
import sys, warnings, numpy as np; sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
dims = tuple(int(v) for v in sys.argv[2].split(","))
g = P.build_cantilever(*dims)
op = P.FineOperator(g, P.simp_modulus(P.make_state("random_floor", *dims, vf=0.5, seed=42), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, sys.argv[3])
r = P.SplitMix64(7).gaussian(g.n_free)
np.save(sys.argv[1], h.vcycle(r))
'''
envs = {"default": {}, "notb": {"SG_ST64_NOTB": "1"}, "st64_unfused": {"SG_ST64_UNFUSED": "1"},
        "p32_unfused": {"SG_P32_UNFUSED": "1"}, "all_unfused": {"SG_P32_UNFUSED": "1", "SG_ST64_UNFUSED": "1"}}
for dims, pol in [tuple(a.split(":")) for a in (sys.argv[1:] or ["64,48,40:fp32", "64,48,40:fp64", "16,8,8:fp32"])]:
    out = {}
    for name, env in envs.items():
        path = f"/tmp/ab_{name}.npy"
        subprocess.run([sys.executable, "-c", code, path, dims, pol], check=True, env=dict(os.environ, **env))
        out[name] = np.load(path)
    base = out["all_unfused"]
    print(dims, pol, {k: (bool(np.array_equal(v, base)), float(np.abs(v - base).max())) for k, v in out.items()})
