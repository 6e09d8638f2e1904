# rz_pupd_z32 experiment (not kept, DESIGN 6b; SG_RZP_ELEM no longer exists): p update one thread per node vs per DOF
O=gpurun_out/r3i.txt
: > $O
for rep in 1 2; do
  for e in 0 1; do
    if [ $e = 1 ]; then export SG_RZP_ELEM=1; else unset SG_RZP_ELEM; fi
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   ELEM=$e solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'])" >> $O
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:rz_pupd --csv \
        --log-file gpurun_out/r3i_$e.csv python tools/solve_launches.py 100 > /dev/null 2>&1
    python tools/launch_summary.py gpurun_out/r3i_$e.csv | head -3 | sed "s/^/   ELEM=$e /" >> $O
  done
done
unset SG_RZP_ELEM
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_behaviour_gpu.py -q -p no:cacheprovider -k "pcg or headline or outer" 2>&1 | tail -1 >> $O
rm -f gpurun_out/r3i_*.csv
