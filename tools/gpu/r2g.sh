timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.txt
SG_HIST_REPORT=1 timeout 600 python -m pytest tests/test_baseline_configs_gpu.py -m gpu -q -s -k "fp32_sweep or jacobi or big_hier" > gpurun_out/hist_report.txt 2>&1
