rm -rf gpurun_out/ncu; mkdir -p gpurun_out/ncu
NCU_KERNELS="fine_pk_kernel<1 fine_pk_kernel<2 fine_p64_kernel stencil_sym_kernel pq_step rz_pupd_z32 prolong_kernel restrict_kernel cheb_first0_p32" bash tools/gpu/ncu_hot.sh
python tools/kernel_times.py 100 > gpurun_out/kernel_times.txt 2>&1
