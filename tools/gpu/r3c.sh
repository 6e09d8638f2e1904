# plain P32 apply: layer loop unrolled by two (PK_Y only) vs not; then the -m gpu suite
O=gpurun_out/r3c.txt
: > $O
L=paper_2604_26441_b200/_lib
for rep in 1 2; do
  for v in nounroll unroll; do
    cp $L/variants/libsg_$v.so $L/libsg_b200.so
    for N in 100 200 64; do
      echo "== $v N=$N $(timeout 300 python tools/pk_kernels.py $N 20 2>&1 | tr '\n' ';')" >> $O
    done
  done
done
cp $L/variants/libsg_unroll.so $L/libsg_b200.so
timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r3c_bench.json
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3c_pytest.txt 2>&1
tail -3 gpurun_out/r3c_pytest.txt >> $O
