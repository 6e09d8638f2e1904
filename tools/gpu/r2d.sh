SG_NVCC_EXTRA=-DSG_TRACE_CLOCK python -c "from paper_2604_26441_b200 import build; build.build()" > gpurun_out/build_clock.txt 2>&1
SG_TRACE_CLOCK=1 python tools/pcg80_trace2.py > gpurun_out/pcg80_trace_clock.txt 2>&1
SG_PCG80_PIPE=1 SG_TRACE_CLOCK=1 python tools/pcg80_trace2.py > gpurun_out/pcg80_trace_clock_pipe.txt 2>&1
