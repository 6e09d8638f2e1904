python tools/env_ab.py SG_SYM_G 0,1,2,3,4,5 100 200 > gpurun_out/symg_ab.txt 2>&1
