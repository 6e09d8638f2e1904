"""Development aid: sweep_axes cell kappa with the symmetric vs full stencil."""
import json, sys
sys.path.insert(0, ".")
from dataclasses import replace
from paper_2604_26441_b200.bench import specs, run_experiment, numeric_payload
g = json.load(open("tests/golden/bench_reports.json"))["sweep_axes"]
ref = json.loads(g["payload"])
over = {k: (tuple(tuple(x) if isinstance(x, list) else x for x in v) if isinstance(v, list) else v) for k, v in g["overrides"].items()}
rep = run_experiment(replace(specs.ExperimentSpec(), **over))
for t, r in zip(rep["trials"], ref["trials"]):
    print(t["levels"], t["degree"], t["restart"], "kappa", t["kappa_eff"], r["kappa_eff"], "it", t["iterations"], r["iterations"])
