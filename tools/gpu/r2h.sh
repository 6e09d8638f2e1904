timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or packed or p32 or fine_apply" > gpurun_out/t_pk.txt 2>&1
python tools/kernel_times.py 100 > gpurun_out/kt.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
bash tools/gpu/ncu_hot.sh
