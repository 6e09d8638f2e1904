"""Development aid: the fused smoother paths must be bit-identical to the
unfused ones.  Runs V-cycles in subprocesses with SG_P32_UNFUSED /
SG_ST64_UNFUSED / SG_NO_P32 and compares the bits."""
import os, subprocess, sys
import numpy as np
code = r'''
import sys, warnings, numpy as np
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
out = {}
for dims, kind, pol, lv in (((16,8,8),"uniform","fp32",4), ((12,12,12),"binary","fp32",4),
                            ((16,16,16),"binary","fp64",4), ((24,16,16),"uniform","fp32",3)):
    g = P.build_cantilever(*dims)
    op = P.FineOperator(g, P.simp_modulus(P.make_state(kind, *dims, vf=0.5, seed=42), 3.0))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, lv, pol)
    r = P.SplitMix64(7).gaussian(g.n_free)
    out[f"{dims}_{kind}_{pol}"] = h.vcycle(r)
    out[f"{dims}_{kind}_{pol}_w"] = h.wcycle(r)
np.savez(sys.argv[1], **{k: v for k, v in out.items()})
'''
open("/tmp/fd_inner.py", "w").write(code)
runs = {"fused": {}, "unfused": {"SG_P32_UNFUSED": "1", "SG_ST64_UNFUSED": "1"},
        "nop32": {"SG_NO_P32": "1", "SG_ST64_UNFUSED": "1"}}
for name, env in runs.items():
    subprocess.run([sys.executable, "/tmp/fd_inner.py", f"/tmp/fd_{name}.npz"], check=True,
                   env=dict(os.environ, **env))
a, b, c = (np.load(f"/tmp/fd_{n}.npz") for n in runs)
for k in a.files:
    print(f"{k:40s} fused==unfused {np.array_equal(a[k], b[k])}  unfused==nop32 {np.array_equal(b[k], c[k])}")
