# block-size A/B of the P32 kernels (SG_PK_NT), then the -m gpu suite at the default
set -x
O=gpurun_out/r3a.txt
: > $O
for rep in 1 2; do
  for nt in 512 256; do
    for N in 100 200; do
      echo "== NT=$nt N=$N $(SG_PK_NT=$nt timeout 300 python tools/pk_kernels.py $N 20 2>&1 | tr '\n' ';')" >> $O
    done
    SG_PK_NT=$nt timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   NT=$nt solve', round(d['value']*1e3,3), d['pcg_iters'], d['final_true_residual'], 'e2e', d['e2e']['value'])" >> $O
  done
done
timeout 600 python tools/env_ab.py SG_PK_NT 512,256 100 200 >> $O 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3a_pytest.txt 2>&1
tail -3 gpurun_out/r3a_pytest.txt >> $O
