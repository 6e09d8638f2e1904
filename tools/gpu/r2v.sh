for rep in 1 2; do
for v in 1184 592 296 148; do
  SG_RED_BLOCKS=$v python bench.py --no-cpu-baseline > gpurun_out/rb_${v}_$rep.json 2>/dev/null
done
done
