L=paper_2604_26441_b200/_lib
cp $L/libsg_b200.so /tmp/keep.so
prof() { python - <<'PY'
import ctypes, sys, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
out = ctypes.c_double()
r = []
for w in (6, 4):
    _native.check(_native.load().sg_hier_profile(h._hh, w, 30, ctypes.byref(out), _dev.stream()))
    r.append(out.value * 1e3)
print("cheb %.2f us  vcycle %.1f us" % tuple(r))
PY
}
for rep in 1 2; do
  for v in head new newxsc; do
    case $v in head) cp $L/variants/libsg_head.so $L/libsg_b200.so; X="";;
               new) cp $L/variants/libsg_new.so $L/libsg_b200.so; X="";;
               newxsc) cp $L/variants/libsg_new.so $L/libsg_b200.so; X=1;; esac
    if [ -n "$X" ]; then export SG_PK_CHEB_XSC=1; else unset SG_PK_CHEB_XSC; fi
    echo "== $v $(prof)" >> gpurun_out/x.txt
    python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'])" >> gpurun_out/x.txt
  done
done
cp /tmp/keep.so $L/libsg_b200.so
