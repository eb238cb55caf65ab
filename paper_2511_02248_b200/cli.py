"""`autoscale` and `sweep` commands with the reference CLI's flags, inputs
and byte-identical outputs (cli.py:46-217, 257-313), planned and placed on
the B200 in batches (runner.py of this package).

    python -m paper_2511_02248_b200.cli autoscale --dag d.json --profiles p.json \\
        --fleet f.json --synth burst:rate=8,duration=600 --mode operator --out out/
    python -m paper_2511_02248_b200.cli sweep ... --sweep seqlen --range 1024,2048,4096

Exit codes: 0 all points feasible, 2 some point violated its SLO, 1
configuration or input error. Profile fitting (`fit`) is not part of the
planner hot path and is not provided.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

from . import errors, model, runner, workload

BUNDLED_DIR = Path(__file__).parent / "data"
TRACE_HEADER = ["timestamp_s", "input_tokens", "output_tokens"]


# --------------------------------------------------------------------------
# input formats (opgraph.py:151-177, perfmodel.py load_profiles,
# placement.py:120-132, workload.py:61-95)


def load_dag(path):
    with open(path, "r", encoding="utf-8") as fh:
        return model.build_dag(json.load(fh))


def load_profiles(path):
    with open(path, "r", encoding="utf-8") as fh:
        return model.profiles_from_dict(json.load(fh))


def load_fleet(path):
    with open(path, "r", encoding="utf-8") as fh:
        raw = json.load(fh)
    return [model.DeviceSpec(id=d["id"], mem_cap=float(d.get("mem_cap", 80e9)),
                             compute_cap=float(d.get("compute_cap", 1.0)),
                             link_bw=float(d.get("link_bw", 600e9))) for d in raw]


def load_trace(path, fmt="csv"):
    """Records sorted (stably) by arrival time, with the reference's checks."""
    if fmt != "csv":
        raise errors.ParseError(f"unsupported trace format {fmt!r}")
    records = []
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None:
            raise errors.EmptyTrace(f"{path}: file is empty")
        if [h.strip() for h in header] != TRACE_HEADER:
            raise errors.ParseError(f"{path}:1: expected header {','.join(TRACE_HEADER)}, "
                                    f"got {','.join(header)}")
        for lineno, row in enumerate(reader, start=2):
            if not row or all(not cell.strip() for cell in row):
                continue
            if len(row) != 3:
                raise errors.ParseError(f"{path}:{lineno}: expected 3 fields, got {len(row)}")
            try:
                t, inp, out = float(row[0]), int(row[1]), int(row[2])
            except ValueError as exc:
                raise errors.ParseError(f"{path}:{lineno}: {exc}") from None
            if t < 0:
                raise errors.ParseError(f"{path}:{lineno}: negative timestamp {t}")
            if inp < 1:
                raise errors.ParseError(f"{path}:{lineno}: input_tokens must be >= 1, got {inp}")
            if out < 0:
                raise errors.ParseError(f"{path}:{lineno}: output_tokens must be >= 0, got {out}")
            records.append(workload.RequestRecord(t, inp, out))
    if not records:
        raise errors.EmptyTrace(f"{path}: no data rows")
    records.sort(key=lambda r: r.arrival_time)
    return records


_SYNTH_KEYS = {
    "rate": ("rate", float), "duration": ("duration", float),
    "seqlen": ("input_len_median", float), "input_median": ("input_len_median", float),
    "input_sigma": ("input_len_sigma", float), "output_median": ("output_len_median", float),
    "output_sigma": ("output_len_sigma", float), "amplitude": ("amplitude", float),
    "period": ("period", float), "burst_factor": ("burst_factor", float),
    "burst_duty": ("burst_duty", float),
}


def parse_synth(text):
    """'kind:key=value,...' synth specs (cli.py:46-80)."""
    kind, _, rest = text.partition(":")
    kwargs = {}
    if rest:
        for pair in rest.split(","):
            key, sep, value = pair.partition("=")
            if not sep:
                raise errors.OpscalerError(f"--synth: expected key=value, got {pair!r}")
            kwargs[key.strip()] = value.strip()
    spec = {}
    for key, value in kwargs.items():
        if key not in _SYNTH_KEYS:
            raise errors.OpscalerError(f"--synth: unknown key {key!r}")
        name, cast = _SYNTH_KEYS[key]
        spec[name] = cast(value)
    if "seqlen" in kwargs and "input_sigma" not in kwargs:
        spec["input_len_sigma"] = 0.0
    try:
        return workload.SynthSpec(kind=kind or "constant", **spec)
    except (TypeError, ValueError) as exc:
        raise errors.OpscalerError(f"--synth: {exc}") from None


def _resolve(path, kind):
    p = Path(path)
    if p.exists():
        return p
    b = BUNDLED_DIR / path
    if b.exists():
        return b
    raise errors.OpscalerError(f"--{kind}: no such file or bundled asset: {path}")


def load_scenario(args):
    dag = load_dag(_resolve(args.dag, "dag"))
    profiles = load_profiles(_resolve(args.profiles, "profiles"))
    fleet = load_fleet(_resolve(args.fleet, "fleet"))
    profiles.validate_against(dag)
    return dag, profiles, fleet


def workload_points(args):
    if bool(args.trace) == bool(args.synth):
        raise errors.OpscalerError("exactly one of --trace or --synth is required")
    if args.trace:
        records = load_trace(_resolve(args.trace, "trace"))
    else:
        records = workload.synth_workload(parse_synth(args.synth), args.seed)
        if not records:
            raise errors.OpscalerError("--synth: generated an empty trace")
    return workload.windowize(records, window_len=args.window_len, quantile=args.quantile)


def phase_params(args, phase, cls=model.AutoscaleParams, err=errors):
    slo = args.slo_prefill if phase == "prefill" else args.slo_decode
    try:
        return cls(slo=slo, epsilon=args.epsilon)
    except ValueError as exc:
        flag = "--slo-prefill" if phase == "prefill" else "--slo-decode"
        raise err.OpscalerError(f"{flag}/--epsilon: {exc}") from None


# --------------------------------------------------------------------------
# commands


def cmd_autoscale(args):
    dag, profiles, fleet = load_scenario(args)
    windows = workload_points(args)
    return runner.autoscale_windows(dag, profiles, fleet, windows, args.mode, args.placement,
                                    lambda ph: phase_params(args, ph), args.out)


def cmd_sweep(args):
    dag, profiles, fleet = load_scenario(args)
    if not args.sweep:
        raise errors.OpscalerError("--sweep: a sweep axis is required")
    if not args.range:
        raise errors.OpscalerError("--range: comma-separated axis values are required")
    if not args.synth:
        raise errors.OpscalerError("--synth: sweeps take their base point from a synth spec")
    try:
        values = [float(v) for v in args.range.split(",") if v.strip()]
    except ValueError as exc:
        raise errors.OpscalerError(f"--range: {exc}") from None
    spec = parse_synth(args.synth)
    base = model.WorkloadPoint(qps=spec.rate, seq_len=max(1, int(spec.input_len_median)), phase="prefill")
    rows = runner.sweep(args.sweep, values, dag, profiles, fleet, base, phase_params(args, "prefill"),
                        placement_mode=args.placement)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    (out / f"sweep_{args.sweep}.csv").write_text(runner.sweep_rows_to_csv(rows))
    return 2 if any(not (r.feasible_baseline and r.feasible_candidate) for r in rows) else 0


def build_parser():
    parser = argparse.ArgumentParser(prog="opscale-b200",
                                     description="Operator-level autoscaling and placement planner (B200)")
    sub = parser.add_subparsers(dest="command", required=True)

    def scenario_flags(p):
        p.add_argument("--dag", required=True, help="DAG spec JSON")
        p.add_argument("--profiles", required=True, help="profile pack JSON")
        p.add_argument("--fleet", required=True, help="fleet config JSON")
        p.add_argument("--slo-prefill", type=float, default=0.5, help="TTFT SLO, seconds")
        p.add_argument("--slo-decode", type=float, default=0.05, help="TBT SLO, seconds")
        p.add_argument("--epsilon", type=float, default=0.0, help="SLO slack buffer, seconds")
        p.add_argument("--placement", choices=("shared", "default_stream"), default="shared")
        p.add_argument("--trace", help="request trace CSV")
        p.add_argument("--synth", help="synthetic workload, e.g. constant:rate=30,seqlen=4096")
        p.add_argument("--out", required=True, help="output directory")
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--window-len", type=float, default=60.0)
        p.add_argument("--quantile", type=float, default=0.95)

    p = sub.add_parser("autoscale", help="plan and place each workload window")
    scenario_flags(p)
    p.add_argument("--mode", choices=("operator", "model", "oracle"), default="operator")
    p = sub.add_parser("sweep", help="savings sweep across one axis")
    scenario_flags(p)
    p.add_argument("--sweep", choices=("seqlen", "qps", "model_scale"), required=True)
    p.add_argument("--range", required=True, help="comma-separated axis values")
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return cmd_autoscale(args) if args.command == "autoscale" else cmd_sweep(args)
    except (errors.OpscalerError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
