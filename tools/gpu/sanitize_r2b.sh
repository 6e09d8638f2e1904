# compute-sanitizer over the kernels added later in round 2: the FP64 block-form
# apply (sg_fine_p64.cu), the record-fed BF16 tcgen05 apply (sg_fine_tc2.cu), the
# device fixtures (sg_fixtures.cu), the vectorised P32 epilogues, the V-cycle /
# PCG paths without the f64 iterate and z (cycle_run_noz, rz_pupd_z32) and the
# peer slab transport (memcheck, two processes).  Summaries -> gpurun_out/san2_<tool>.txt
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_parity.py tests/test_fixtures_gpu.py"
K="(fp64_block_tiling or fp64_general_mask or bf16_tiling or bf16_general_mask or fused_smoothers or outer_solver or hierarchy_and_cycle or device_state or robustness or operator_from_device) and not dims0"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 30 --error-exitcode 0 \
      python -m pytest $SEL -m gpu -q -x -k "$K" -p no:cacheprovider \
      > gpurun_out/san2_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san2_rc.txt
done
SLAB_TRANSPORT=peer timeout 1500 $CS --tool memcheck --target-processes all --print-limit 30 \
    --error-exitcode 0 python -m pytest tests/test_slab_gpu.py -m gpu -q -x -k "2-peer" \
    -p no:cacheprovider > gpurun_out/san2_memcheck_slab.txt 2>&1
