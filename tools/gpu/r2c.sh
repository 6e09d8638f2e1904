timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pcg80" > gpurun_out/t_pcg80.txt 2>&1
python tools/pcg80_trace2.py > gpurun_out/pcg80_trace.txt 2>&1
python tools/pcg80_probe.py > gpurun_out/pcg80_probe.txt 2>&1
SG_PCG80_PIPE=1 python tools/pcg80_probe.py > gpurun_out/pcg80_probe_pipe.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
