set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=40 > gpurun_out/gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
