# Round-end validation on one B200: GPU tests, smoke, both bench arms, 200^3 bench.
python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --size 200 --steps 5 --warmup 3 > gpurun_out/final_bench200.json 2> gpurun_out/final_bench200.err
