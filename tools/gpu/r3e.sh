# layer-loop unroll by two extended to the fused residual ("res") and to every
# mode incl. the fused smoother ("all", spills 108 B) vs HEAD (plain apply only)
O=gpurun_out/r3e.txt
: > $O
L=paper_2604_26441_b200/_lib
for rep in 1 2; do
  for v in head res all; do
    cp $L/variants/libsg_$v.so $L/libsg_b200.so
    echo "== $v N=100 $(timeout 300 python tools/pk_kernels.py 100 20 2>&1 | tr '\n' ';')" >> $O
    echo "== $v N=200 $(timeout 300 python tools/pk_kernels.py 200 20 2>&1 | tr '\n' ';')" >> $O
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   $v solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'])" >> $O
  done
done
for v in res all; do
  cp $L/variants/libsg_$v.so $L/libsg_b200.so
  echo "-- tests $v" >> $O
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fused or block_size or fine_apply_fp32 or vcycle" 2>&1 | tail -1 >> $O
done
cp $L/variants/libsg_head.so $L/libsg_b200.so
