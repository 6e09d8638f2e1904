SG_HIST_REPORT=1 timeout 1200 python -m pytest tests/test_baseline_configs_gpu.py -m gpu -q -s -rA --durations=60 > gpurun_out/hist_report.txt 2>&1
python tools/pcg80_trace2.py > gpurun_out/pcg80_trace.txt 2>&1
python tools/pcg80_probe.py > gpurun_out/pcg80_probe.txt 2>&1
