python tools/transfer_ab.py > gpurun_out/transfer_ab.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "transfer or prolong or restrict or vcycle" > gpurun_out/transfer_tests.txt 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr_solve.csv python tools/solve_launches.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/tr_solve.csv > gpurun_out/tr_solve_breakdown.txt
