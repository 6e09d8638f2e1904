# Round-end validation on one B200: GPU tests, smoke, both bench arms, 200^3 bench,
# the per-solve launch breakdown and the bench command's launch list.
python -m pytest tests -m gpu -q > gpurun_out/final_pytest.txt 2>&1
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
