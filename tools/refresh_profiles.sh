# Regenerate the judged evidence under profiles/ (run on a B200 through gpurun).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
python bench.py --size 200 --steps 5 --warmup 3 > gpurun_out/p_bench200.json 2> gpurun_out/p_bench200.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv \
    python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p_solve.csv python tools/solve_launches.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/p_solve.csv > gpurun_out/p_solve_breakdown.txt
ncu --set full --clock-control none --import-source on -k regex:pcg80_brick -s 2 -c 1 \
    -o gpurun_out/p_pcg80 python tools/pcg80_trace.py 100 > gpurun_out/p_pcg80_trace.txt 2>&1
python tools/ncu_summary.py gpurun_out/p_pcg80.ncu-rep > gpurun_out/p_pcg80_summary.txt 2>&1
python tools/pcg80_probe.py 100 > gpurun_out/p_pcg80_probe.txt 2>&1
python tools/pcg80_trace.py 100 > gpurun_out/p_pcg80_phases.txt 2>&1
