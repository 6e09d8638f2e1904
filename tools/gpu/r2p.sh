for i in 1 2; do
python bench.py --no-cpu-baseline > gpurun_out/fb_new_$i.json 2>/dev/null
SG_PCG_FENCE_BAR=1 python bench.py --no-cpu-baseline > gpurun_out/fb_old_$i.json 2>/dev/null
done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fb_solve.csv python tools/solve_launches.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/fb_solve.csv > gpurun_out/fb_solve_breakdown.txt
python -m pytest tests -m gpu -q -x -k "fused or slab or pcg" > gpurun_out/fb_tests.txt 2>&1
