mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fine_p64 -c 1 -o gpurun_out/ncu/p64src python tools/solve_launches.py 100 > /dev/null 2>&1
ncu -i gpurun_out/ncu/p64src.ncu-rep --page raw --csv > gpurun_out/ncu_p64_raw.csv 2>&1
ncu -i gpurun_out/ncu/p64src.ncu-rep --page source --csv > gpurun_out/ncu_p64_src.csv 2>&1
ncu -i gpurun_out/ncu/p64src.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_p64_cuda.csv 2>&1
