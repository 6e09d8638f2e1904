L=paper_2604_26441_b200/_lib
cp $L/libsg_b200.so /tmp/keep.so
for rep in 1 2; do
for v in rz1 rz2 rz4; do
  cp $L/variants/libsg_$v.so $L/libsg_b200.so
  python bench.py --no-cpu-baseline > gpurun_out/w_${v}_$rep.json 2>/dev/null
done
done
cp $L/variants/libsg_rz4.so $L/libsg_b200.so
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w_solve.csv python tools/solve_launches.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/w_solve.csv > gpurun_out/w_breakdown.txt
cp /tmp/keep.so $L/libsg_b200.so
