# ncu --set full of the hot kernels of one 100^3 FP32-GMG solve (and the plain
# P32 apply, which the solve does not launch: tools/kernel_times.py)
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$NCU -k regex:fine_pk_kernel.0 -c 1 -o gpurun_out/ncu/pk0 python tools/kernel_times.py 100 > /dev/null 2>&1
for k in ${NCU_KERNELS:-"fine_pk_kernel<1" "fine_pk_kernel<2" "fine_apply_walsh_kernel<double" "stencil_sym_kernel" "prolong_kernel" "restrict_kernel" "pq_step" "rz_pupd" "cheb_first0_p32"}; do
  n=$(echo "$k" | tr -c 'a-z0-9_\n' '_')
  $NCU --profile-from-start off -k "regex:$k" -c 1 -o gpurun_out/ncu/$n python tools/solve_launches.py 100 > /dev/null 2>&1
done
for f in gpurun_out/ncu/*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/ncu_hot_summary.txt 2>&1
