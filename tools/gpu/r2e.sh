timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pcg80" > gpurun_out/t_pcg80.txt 2>&1
python tools/pcg80_probe.py > gpurun_out/pcg80_probe.txt 2>&1
SG_NVCC_EXTRA=-DSG_TRACE_CLOCK python -c "from paper_2604_26441_b200 import build; build.build()" > gpurun_out/build_clock.txt 2>&1
SG_TRACE_CLOCK=1 timeout 300 python tools/pcg80_trace2.py > gpurun_out/pcg80_trace_clock.txt 2>&1
