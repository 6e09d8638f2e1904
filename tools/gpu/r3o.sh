# the reference-facing CLI at round-end HEAD (GPU-backed): validate gates, robustness, one timed solve
O=gpurun_out/o_cli.txt
{ echo "# python -m paper_2604_26441_b200 validate"; timeout 600 python -m paper_2604_26441_b200 validate --out gpurun_out/o_validate.json 2>&1 | tail -40;
  echo "# python -m paper_2604_26441_b200 robustness"; timeout 600 python -m paper_2604_26441_b200 robustness --out gpurun_out/o_robustness.json 2>&1 | tail -30;
  echo "# python -m paper_2604_26441_b200 solve --grid 100,100,100 --precision fp32 --trials 3"; timeout 600 python -m paper_2604_26441_b200 solve --grid 100,100,100 --precision fp32 --trials 3 2>&1 | tail -15; } > $O
