set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/gputest.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
