mkdir -p gpurun_out/ncu
cat > /tmp/p0.py <<'PY'
import ctypes, sys, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32", coarse_pcg_steps=0)
out = ctypes.c_double()
_native.check(_native.load().sg_hier_profile(h._hh, 9, 3, ctypes.byref(out), _dev.stream()))
PY
ncu --set full --clock-control none --import-source on -k regex:pcg80_brick -c 3 -o gpurun_out/ncu/p0 python /tmp/p0.py > gpurun_out/p0.log 2>&1
ncu -i gpurun_out/ncu/p0.ncu-rep --page raw --csv > gpurun_out/p0_raw.csv 2>&1
ncu -i gpurun_out/ncu/p0.ncu-rep --page source --csv > gpurun_out/p0_src.csv 2>&1
