# P32 kernels with the products that feed additions as scalar mul.rn (no ptxas
# FFMA2 contraction): alone ("fix") and with the plain apply's layer loop
# unrolled by two ("fixunroll", the candidate), against HEAD ("nounroll");
# then the -m gpu suite and the bench line on the candidate
O=gpurun_out/r3d.txt
: > $O
L=paper_2604_26441_b200/_lib
for rep in 1 2; do
  for v in nounroll fix fixunroll; do
    cp $L/variants/libsg_$v.so $L/libsg_b200.so
    for N in 100 200; do
      echo "== $v N=$N $(timeout 300 python tools/pk_kernels.py $N 20 2>&1 | tr '\n' ';')" >> $O
    done
  done
done
cp $L/variants/libsg_fixunroll.so $L/libsg_b200.so
timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r3d_bench.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3d_pytest.txt 2>&1
tail -3 gpurun_out/r3d_pytest.txt >> $O
