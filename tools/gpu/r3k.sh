# pcg80 merged-collect experiment (not kept, DESIGN 6b; the variant library was built from a working-tree change)
# block barrier fewer per step) vs HEAD; then the -m gpu suite on merged
O=gpurun_out/r3k.txt
: > $O
L=paper_2604_26441_b200/_lib
for rep in 1 2; do
  for v in head merged; do
    cp $L/variants/libsg_$v.so $L/libsg_b200.so
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   $v solve', round(d['value']*1e3,3), 'pcg80', round(d['components']['coarsest_pcg80']['ms']*1e3,1), 'us', d['pcg_iters'], d['final_true_residual'])" >> $O
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:pcg80 --csv \
        --log-file gpurun_out/r3k_$v.csv python tools/solve_launches.py 100 > /dev/null 2>&1
    python tools/launch_summary.py gpurun_out/r3k_$v.csv | head -2 | tail -1 | sed "s/^/   $v ncu /" >> $O
  done
done
cp $L/variants/libsg_merged.so $L/libsg_b200.so
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3k_pytest.txt 2>&1
tail -2 gpurun_out/r3k_pytest.txt >> $O
rm -f gpurun_out/r3k_*.csv
