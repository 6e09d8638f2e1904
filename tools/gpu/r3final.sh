# Round-end validation and evidence at HEAD (one B200): GPU tests, smoke, both
# bench arms, 200^3 bench, per-solve launch breakdown, bench launch list, and
# ncu --set full of the kernels whose tiling changed (fused P32 applies, FP64 apply).
mkdir -p gpurun_out/ncu
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --size 200 --steps 5 --warmup 3 > gpurun_out/final_bench200.json 2> gpurun_out/final_bench200.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final_solve.csv python tools/solve_launches.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/final_solve.csv > gpurun_out/final_solve_breakdown.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/final_launches.csv > gpurun_out/final_launches_summary.txt
NCU="ncu --set full --clock-control none --import-source on"
# the four level-0 applies (plain, fused smoother, fused residual, FP64) of tools/pk_kernels.py
$NCU --profile-from-start off -k regex:fine_p -c 4 -o gpurun_out/ncu/fine_level0 python tools/pk_kernels.py 100 > gpurun_out/final_pk_ncu.log 2>&1
for f in gpurun_out/ncu/*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/final_ncu_summary.txt 2>&1
rm -f gpurun_out/final_solve.csv
