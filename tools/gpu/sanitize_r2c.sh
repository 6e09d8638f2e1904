# compute-sanitizer over the cooperative PCG kernels with the release/acquire
# grid barrier and the pinned-staging input path (round-end HEAD).
CS=/usr/local/cuda/bin/compute-sanitizer
K="outer_solver or fused_pcg or numpy_inputs or headline or pcg"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 30 --error-exitcode 0 \
      python -m pytest tests/test_gpu_parity.py tests/test_reference_behaviour_gpu.py -m gpu -q -x -k "$K" \
      -p no:cacheprovider > gpurun_out/san3_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san3_rc.txt
done
