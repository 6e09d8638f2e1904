"""Development aid: per-phase timing of one pcg80 step for every block (%globaltimer)."""
import ctypes, sys, warnings
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
for rep in range(3):
    t = np.zeros(64 * 256, dtype=np.int64)  # sg_hier_pcg80_trace writes 8 steps x 8 stamps per block
    _native.check(lib.sg_hier_pcg80_trace(h._hh, t.ctypes.data, _dev.stream()))
    t = t.reshape(256, 8, 8)[:, 0, :]  # step 8 of every block
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    # stamps (brick kernel): 0 step start, 5 window staged, 1 phase A done, 2 pq known, 3 phase B done, 4 rzn known
    for k, name in enumerate(["start", "A_done", "pq_out", "B_done", "rz_out", "fill_done", "s6", "s7"]):
        col = rel[:, k]
        print(f"{name:7s} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f} us "
              f"(argmax blk {int(col.argmax())})")
    print("blocks", len(t))
