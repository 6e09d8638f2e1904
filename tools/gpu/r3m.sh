# pcg80 at round-end HEAD: ncu --set full of one coarsest solve + the per-step phase trace
ncu --set full --clock-control none --import-source on -k regex:pcg80_brick -s 2 -c 1 \
    -o gpurun_out/m_pcg80 python tools/pcg80_trace.py 100 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/m_pcg80.ncu-rep > gpurun_out/m_pcg80_summary.txt 2>&1
python tools/pcg80_trace.py 100 > gpurun_out/m_pcg80_phases.txt 2>&1
