# cluster residency probe; FP64 apply block-size A/B (SG_P64_NT); solve with the
# new P32 defaults; block-size bit-identity tests
O=gpurun_out/r3b.txt
: > $O
./tools/micro/cluster_occ >> $O 2>&1
for rep in 1 2; do
  for nt in 512 256; do
    for N in 100 200; do
      echo "== P64_NT=$nt N=$N $(SG_P64_NT=$nt timeout 300 python tools/pk_kernels.py $N 20 2>&1 | tr '\n' ';')" >> $O
    done
    SG_P64_NT=$nt timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   P64_NT=$nt solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'], 'e2e', d['e2e']['value'])" >> $O
  done
done
for N in 80 40; do
  for nt in 512 256; do
    echo "== PK_NT=$nt N=$N $(SG_PK_NT=$nt timeout 300 python tools/pk_kernels.py $N 20 2>&1 | tr '\n' ';')" >> $O
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "block_size or fp64 or p32 or fine_apply" >> $O 2>&1
