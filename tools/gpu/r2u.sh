L=paper_2604_26441_b200/_lib
cp $L/libsg_b200.so /tmp/keep.so
for v in head new head new; do
  cp $L/variants/libsg_$v.so $L/libsg_b200.so
  echo "== $v" >> gpurun_out/u.txt
  python tools/pcg80_launch_probe.py 100 >> gpurun_out/u.txt 2>&1
done
cp /tmp/keep.so $L/libsg_b200.so
python -m pytest tests -m gpu -q -x -k "pcg80 or coarsest or headline or vcycle" > gpurun_out/u_tests.txt 2>&1
