for e in "SG_PCG80_PIPE=1" "SG_PCG80_PIPE=1 SG_PCG80_NREP=4" "SG_PCG80_PIPE=1 SG_PCG80_NREP=8" "SG_PCG80_PIPE=1 SG_PCG80_NREP=16"; do
  echo "== $e" >> gpurun_out/pcg80_sweep.txt
  env $e python tools/pcg80_probe.py 2>&1 | tail -2 >> gpurun_out/pcg80_sweep.txt
done
SG_PCG80_PIPE=1 SG_PCG80_NREP=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pcg80" > gpurun_out/t_pcg80.txt 2>&1
