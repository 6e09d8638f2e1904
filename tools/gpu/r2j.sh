python tools/pk_kernels.py 100 20 > gpurun_out/pk_times.txt 2>&1
mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fine_pk|walsh" -c 4 -o gpurun_out/ncu/l0 python tools/pk_kernels.py 100 1 > gpurun_out/ncu_l0.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu/l0.ncu-rep > gpurun_out/ncu_l0_summary.txt 2>&1
