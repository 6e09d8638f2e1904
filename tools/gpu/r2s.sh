# FP64 apply A/B across library builds (variants/ copied over the in-tree .so)
L=paper_2604_26441_b200/_lib
cp $L/libsg_b200.so /tmp/keep.so
for v in ${VARS:-head new head new}; do
  cp $L/variants/libsg_$v.so $L/libsg_b200.so
  echo "== $v" >> gpurun_out/p64_var.txt
  python tools/p64_ab.py SG_P64_RTNT - >> gpurun_out/p64_var.txt 2>&1
  python -c "import hashlib,numpy as np; print('sha', hashlib.sha1(np.load('/tmp/p64ab.npy').tobytes()).hexdigest())" >> gpurun_out/p64_var.txt
done
cp /tmp/keep.so $L/libsg_b200.so
