import os, sys, warnings, subprocess
sys.path.insert(0, ".")
import numpy as np
code = r'''
import sys, warnings, numpy as np
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
for dims, kind in (((16,8,8),"uniform"), ((12,12,12),"binary")):
    g = P.build_cantilever(*dims)
    op = P.FineOperator(g, P.simp_modulus(P.make_state(kind, *dims, vf=0.5, seed=42), 3.0))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, "fp32")
    r = P.SplitMix64(7).gaussian(g.n_free)
    np.save(f"/tmp/v_{dims[0]}_{kind}_{sys.argv[1]}.npy", h.vcycle(r))
'''
open("/tmp/diag_inner.py","w").write(code)
subprocess.run([sys.executable, "/tmp/diag_inner.py", "p32"], check=True)
subprocess.run([sys.executable, "/tmp/diag_inner.py", "nop32"], check=True, env=dict(os.environ, SG_NO_P32="1"))
subprocess.run([sys.executable, "/tmp/diag_inner.py", "unf"], check=True, env=dict(os.environ, SG_P32_UNFUSED="1"))
for dims, kind in (((16,8,8),"uniform"), ((12,12,12),"binary")):
    a = np.load(f"/tmp/v_{dims[0]}_{kind}_p32.npy"); b = np.load(f"/tmp/v_{dims[0]}_{kind}_nop32.npy")
    c = np.load(f"/tmp/v_{dims[0]}_{kind}_unf.npy")
    print(dims, kind, "p32 vs nop32", np.array_equal(a, b), np.linalg.norm(a-b)/np.linalg.norm(b),
          "unfused vs nop32", np.array_equal(c, b), "fused vs unfused", np.array_equal(a, c))
