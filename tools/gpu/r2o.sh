mkdir -p gpurun_out/ncu
for k in pq_step rz_pupd_z32; do
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -s 2 -c 1 -o gpurun_out/ncu/$k python tools/solve_launches.py 100 > gpurun_out/ncu_$k.log 2>&1
ncu -i gpurun_out/ncu/$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>&1
ncu -i gpurun_out/ncu/$k.ncu-rep --page source --csv > gpurun_out/ncu_${k}_src.csv 2>&1
done
