# plain P32 apply (unrolled) with 512- vs 256-thread blocks (SG_PK_NT forces every mode)
O=gpurun_out/r3j.txt
: > $O
for rep in 1 2; do
  for nt in 512 256; do
    for N in 100 80 200; do
      echo "== NT=$nt N=$N $(SG_PK_NT=$nt timeout 300 python tools/pk_kernels.py $N 20 2>&1 | head -1)" >> $O
    done
  done
done
