"""Command-line front end: ``python -m paper_2604_26441_b200 {validate,solve,sweep,probe,robustness}``.

Same sub-commands, flags and exit codes as the reference CLI (simpgmg/cli.py:32-147):
0 = every gate passed, 1 = a gate failed, 2 = the options do not form a valid
experiment spec.  ``--out`` writes the 17-digit JSON report.
"""

from __future__ import annotations

import argparse
import sys

from .bench.specs import (METHODS, PRECISIONS, SMOOTHERS, STATE_KINDS, make_spec, parse_grid)


def _csv(conv):
    return lambda text: tuple(conv(t.strip()) for t in text.split(",") if t.strip())


# (flag, dest in single-cell mode, dest in sweep mode, single parser, sweep parser, choices)
_AXES = (
    ("--grid", "grid", "grids", parse_grid, parse_grid, None),
    ("--vf", "vf", "vfs", float, _csv(float), None),
    ("--p", "p", "ps", float, _csv(float), None),
    ("--smoother", "smoother", "smoothers", str, _csv(str), SMOOTHERS),
    ("--degree", "degree", "degrees", int, _csv(int), None),
    ("--levels", "levels", "depths", int, _csv(int), None),
    ("--restart", "restart", "restarts", int, _csv(int), None),
    ("--precision", "precision", "precisions", str, _csv(str), PRECISIONS),
)
_SCALARS = (("--floor", float), ("--alpha", float), ("--seed", int), ("--tol", float),
            ("--maxiter", int), ("--trials", int), ("--warmups", int))
_HELP = {
    "validate": "run the M1-M8 correctness gates",
    "solve": "repeated timed solves of one configuration",
    "sweep": "grid x vf x p (x smoother/degree/depth/restart/precision) cartesian sweep",
    "probe": "Lanczos kappa_eff probe of the FP64 V-cycle preconditioned operator",
    "robustness": "ten adversarial density states through FGMRES",
}


def _options(p: argparse.ArgumentParser, sweep: bool) -> None:
    p.add_argument("--config", help="key = value config file")
    for flag, single, multi, conv1, convn, choices in _AXES:
        if sweep:
            kw = {"action": "append"} if flag == "--grid" else {}
            p.add_argument(flag, dest=multi, type=convn, **kw)
        else:
            p.add_argument(flag, dest=single, type=conv1, choices=choices)
    p.add_argument("--state", choices=STATE_KINDS)
    p.add_argument("--method", choices=METHODS)
    for flag, conv in _SCALARS:
        p.add_argument(flag, type=conv)
    p.add_argument("--out", help="write the structured report to this file")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2604_26441_b200",
                                 description="GMG-preconditioned Krylov experiments on B200")
    sub = ap.add_subparsers(dest="experiment", required=True)
    for name, text in _HELP.items():
        sp = sub.add_parser(name, help=text)
        _options(sp, sweep=(name == "sweep"))
        if name == "robustness":
            sp.set_defaults(restart=50, maxiter=500)
    return ap


def _summary(report: dict) -> str:
    spec = report["spec"]
    lines = [f"{spec['experiment']}: grid {spec['grid']} precision {spec['precision']}"]
    for key, val in report.get("aggregates", {}).items():
        if not isinstance(val, dict):
            lines.append(f"  {key} = {val}")
    for g in report.get("gates", []):
        lines.append(f"  [{'PASS' if g['passed'] else 'FAIL'}] {g['id']}: {g['measured']} "
                     f"(threshold {g['threshold']})")
    return "\n".join(lines)


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    overrides = {k: v for k, v in vars(args).items() if k not in ("experiment", "config", "out")}
    try:
        spec = make_spec(args.experiment, args.config, **overrides)
    except (ValueError, TypeError, OSError) as exc:
        print(f"invalid experiment spec: {exc}", file=sys.stderr)
        return 2
    from .bench.reports import dumps_report
    from .bench.runner import exit_code, run_experiment
    report = run_experiment(spec)
    print(_summary(report))
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(dumps_report(report))
        print(f"report written to {args.out}")
    return exit_code(report)


if __name__ == "__main__":
    sys.exit(main())
