# FP64 apply: new block-form kernel vs the scalar Walsh kernel (SG_WALSH64_OLD=1)
python tools/pk_kernels.py 100 20 2>&1 | grep FP64
SG_WALSH64_OLD=1 python tools/pk_kernels.py 100 20 2>&1 | grep FP64
