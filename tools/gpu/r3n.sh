# symmetric L1 stencil occupancy: __launch_bounds__(128, 4) (head) vs 5 / 6 / 8 blocks per SM
O=gpurun_out/r3n.txt
: > $O
L=paper_2604_26441_b200/_lib
for rep in 1 2; do
  for v in head st5 st6 st8; do
    cp $L/variants/libsg_$v.so $L/libsg_b200.so
    echo "== $v $(timeout 300 python tools/env_ab.py SG_DUMMY_AB x 100 2>&1 | tail -1)" >> $O
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   $v solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'], 'l1', round(d['components']['level1_spmv_fp64']['ms']*1e3,1))" >> $O
  done
done
for v in head st5 st6 st8; do
  cp $L/variants/libsg_$v.so $L/libsg_b200.so
  timeout 300 python tools/env_ab.py SG_DUMMY_AB x 100 > /dev/null 2>&1; cp /tmp/envab_x.npy /tmp/vc_$v.npy
done
python -c "
import numpy as np
a=np.load('/tmp/vc_head.npy')
for v in ('st5','st6','st8'): print('   vcycle bits', v, np.array_equal(a, np.load('/tmp/vc_%s.npy'%v)))" >> $O
cp $L/variants/libsg_head.so $L/libsg_b200.so
