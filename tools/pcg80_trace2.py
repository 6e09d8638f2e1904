"""Development aid: per-phase timing of pcg80 steps 8..15 for every block of the
pipelined brick kernel (%globaltimer stamps; sg_hier_pcg80_trace).
stamps: 0 step start, 1 published (m + partials), 5 halo filled, 3 SpMV done,
6 partial packets validated (warp 0), 2 (gamma, delta) known, 4 update done."""
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
    # PCG80_STEPS=12: steps 12..15 do not run, so trace slot 7 keeps the prologue stamps
    h = P.build_hierarchy(op, 4, "fp32", coarse_pcg_steps=int(os.environ.get("PCG80_STEPS", "80")))
h.vcycle(np.ones(g.n_free))
NAMES = [(0, "start"), (1, "publish"), (5, "fill"), (3, "spmv"), (6, "validate"), (2, "collect"), (4, "update")]
for rep in range(2):
    t = np.zeros(64 * 256, dtype=np.int64)
    _native.check(lib.sg_hier_pcg80_trace(h._hh, t.ctypes.data, _dev.stream()))
    t = t.reshape(256, 8, 8)
    nb = int((t[:, 0, 0] > 0).sum())
    t = t[:nb].astype(np.float64) / (1.965e3 if os.environ.get("SG_TRACE_CLOCK") else 1e3)  # us
    ns = min(8, int(os.environ.get("PCG80_STEPS", "80")) - 8)
    starts = t[:, :ns, 0]
    period = np.diff(starts, axis=1)
    print(f"rep {rep}: blocks {nb}; step period med {np.median(period):.3f} us "
          f"(min {period.min():.3f} max {period.max():.3f}); start skew per step "
          + " ".join(f"{v:.2f}" for v in (starts.max(0) - starts.min(0))))
    prev = 0
    for k, name in NAMES[1:]:
        d = t[:, :ns, k] - t[:, :ns, prev]
        print(f"  {name:9s} med {np.median(d):6.3f}  p90 {np.percentile(d, 90):6.3f}  max {d.max():6.3f} us")
        prev = k
    # global step boundary: first block start to last block start of next step
    # offsets of every stamp from the block's step start, in time order
    # (the early-halo variant stamps 0 start, 3 SpMV, 2 collect, 1 publish, 5 fill, 4 end)
    rel = {k: np.median(t[:, :ns, k] - t[:, :ns, 0]) for k in range(8) if (t[:, :ns, k] > 0).all()}
    print("  offsets: " + ", ".join(f"{k}:{v:.2f}" for k, v in sorted(rel.items(), key=lambda kv: kv[1])))
    # prologue (early-halo variant, slot 15): 0 entry, 1 TMEM allocated, 2 TMEM rows
    # stored, 3 bulk copy landed + fill cells, 4 before the first SpMV, 5 after it, 6 window m0
    p = t[:, 7, :7] - t[:, 7, :1]
    print("  prologue: " + ", ".join(f"{k}:{np.median(p[:, k]):.2f}" for k in range(7)))
    e = t[:, 7, 0]
    s8 = t[:, 0, 0]
    print(f"  entry spread {e.max() - e.min():.2f} us; entry -> step 8 start: med {np.median(s8 - e):.2f} "
          f"(min {np.min(s8 - e):.2f} max {np.max(s8 - e):.2f}); first entry -> last step-15 stamp "
          f"{t[:, ns - 1, 4].max() - e.min():.2f} us")
