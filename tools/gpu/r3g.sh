# clean bench lines at HEAD (no ncu / pytest before them in this process tree)
python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
python bench.py > gpurun_out/g_bench2.json 2> gpurun_out/g_bench2.err
python bench.py --size 200 --steps 5 --warmup 3 > gpurun_out/g_bench200.json 2> gpurun_out/g_bench200.err
nproc > gpurun_out/g_host.txt; uptime >> gpurun_out/g_host.txt
