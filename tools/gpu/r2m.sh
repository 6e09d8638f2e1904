mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stencil_sym_kernel -s 2 -c 1 -o gpurun_out/ncu/sym python tools/solve_launches.py 100 > gpurun_out/ncu_sym.log 2>&1
ncu -i gpurun_out/ncu/sym.ncu-rep --page raw --csv > gpurun_out/ncu_sym_raw.csv 2>&1
ncu -i gpurun_out/ncu/sym.ncu-rep --page source --csv > gpurun_out/ncu_sym_src.csv 2>&1
