python tools/kernel_times.py 100 > gpurun_out/kt.txt 2>&1
NCU_KERNELS='fine_pk_kernel.1 fine_pk_kernel.2 fine_apply_walsh_kernel.double' bash tools/gpu/ncu_hot.sh
