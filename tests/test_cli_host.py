"""Host side of the batched runner / CLI (no GPU): input loaders, synth
specs, windowing, fingerprints and CSV formatting against the reference
CLI's own artifacts (tests/golden/cli.json, make_golden_cli.py)."""

import argparse
import os

import pytest

import golden_cases as G
from paper_2511_02248_b200 import cli, errors, model, runner

IN = os.path.join(os.path.dirname(__file__), "golden", "cli")
CASES = G.load("cli.json")


def _args(argv):
    return cli.build_parser().parse_args(argv + ["--out", "/nonexistent"])


def _in_dir(fn):
    cwd = os.getcwd()
    os.chdir(IN)
    try:
        return fn()
    finally:
        os.chdir(cwd)


@pytest.mark.parametrize("case", [c for c in CASES if c["argv"][0] == "autoscale" and "metrics.csv" in c["texts"]],
                         ids=lambda c: c["name"])
def test_autoscale_rows_prefix_and_fingerprint(case):
    """window / phase / qps / seq_len / mode / placement columns and the
    fingerprint of every metrics.csv row, from this package's windowing."""
    args = _args(case["argv"])
    windows = _in_dir(lambda: cli.workload_points(args))
    lines = case["texts"]["metrics.csv"].splitlines()
    assert lines[0] == runner.METRICS_CSV_HEADER
    rows = lines[1:]
    assert len(rows) == 2 * len(windows)
    for k, (i, point) in enumerate((i, pt) for i, w in enumerate(windows) for pt in w):
        cols = rows[k].split(",")
        assert cols[:7] == [runner.fmt(point.window[0]), runner.fmt(point.window[1]), point.phase,
                            runner.fmt(point.qps) if point.qps > 0 else "0",
                            str(point.seq_len) if point.qps > 0 else "1", args.mode, args.placement]
        if point.qps > 0:
            slo = args.slo_prefill if point.phase == "prefill" else args.slo_decode
            assert cols[-1] == runner.workload_fingerprint(point, slo)
        else:
            assert cols[7:] == ["true", "0", "0", "0", "0", "0", "0", ""]


@pytest.mark.parametrize("case", [c for c in CASES if c["argv"][0] == "sweep"], ids=lambda c: c["name"])
def test_sweep_csv_axis_and_fingerprints(case):
    args = _args(case["argv"])
    text = case["texts"][f"sweep_{args.sweep}.csv"]
    lines = text.splitlines()
    assert lines[0] == runner.SWEEP_CSV_HEADER
    spec = cli.parse_synth(args.synth)
    base = model.WorkloadPoint(qps=spec.rate, seq_len=max(1, int(spec.input_len_median)), phase="prefill")
    values = [float(v) for v in args.range.split(",")]
    for line, v in zip(lines[1:], values):
        cols = line.split(",")
        assert cols[0] == args.sweep and cols[1] == runner.fmt(v)
        pt, slo = base, args.slo_prefill
        if args.sweep == "seqlen":
            scale = v / base.seq_len
            pt = model.WorkloadPoint(qps=base.qps / scale, seq_len=int(v), phase="prefill")
            slo = args.slo_prefill * scale
        elif args.sweep == "qps":
            pt = model.WorkloadPoint(qps=v, seq_len=base.seq_len, phase="prefill")
        if pt.qps <= 0:
            assert cols[2:] == ["0", "0", "0", "true", "true", ""]
        else:
            assert cols[-1] == runner.workload_fingerprint(pt, slo, {"axis": args.sweep, "value": v})


def test_loaders_read_the_cli_inputs():
    dag = cli.load_dag(os.path.join(IN, "dag_70b.json"))
    prof = cli.load_profiles(os.path.join(IN, "profiles_70b.json"))
    prof.validate_against(dag)
    fleet = cli.load_fleet(os.path.join(IN, "fleet_hetero.json"))
    assert len(fleet) == 96 and {d.mem_cap for d in fleet} == {80e9, 40e9, 180e9}
    recs = cli.load_trace(os.path.join(IN, "trace_gap.csv"))
    assert all(a.arrival_time <= b.arrival_time for a, b in zip(recs, recs[1:]))


def test_trace_and_synth_errors(tmp_path):
    bad = tmp_path / "t.csv"
    bad.write_text("t,in,out\n1,2,3\n")
    with pytest.raises(errors.ParseError):
        cli.load_trace(bad)
    bad.write_text("timestamp_s,input_tokens,output_tokens\n1.0,0,3\n")
    with pytest.raises(errors.ParseError):
        cli.load_trace(bad)
    bad.write_text("timestamp_s,input_tokens,output_tokens\n")
    with pytest.raises(errors.EmptyTrace):
        cli.load_trace(bad)
    with pytest.raises(errors.OpscalerError):
        cli.parse_synth("constant:rate")
    with pytest.raises(errors.OpscalerError):
        cli.parse_synth("constant:speed=3")
    assert cli.parse_synth("constant:seqlen=4096").input_len_sigma == 0.0


def test_guard_and_param_errors_before_any_launch(tmp_path, capsys):
    """Cases the reference rejects before planning need no device."""
    for c in CASES:
        if c["name"] not in ("auto_7b_oracle_guard",):
            continue
        rc = _in_dir(lambda: cli.main(c["argv"] + ["--out", str(tmp_path / c["name"])]))
        assert rc == c["exit"]
        assert capsys.readouterr().err == c["stderr"]


def test_fmt_and_compare():
    assert runner.fmt(float("nan")) == "" and runner.fmt(float("inf")) == "inf"
    assert runner.fmt(0.1 + 0.2) == "0.3" and runner.fmt(1e-12) == "1e-12"
    b = runner.ScenarioEval("model/shared", "f", 4, 10.0, 100.0, True)
    c = runner.ScenarioEval("operator/shared", "f", 3, 7.5, 120.0, True)
    r = runner.compare(b, c)
    assert (r.gpu_savings, r.energy_savings, r.memory_savings) == (0.25, 0.25, -0.2)
    with pytest.raises(errors.MismatchedScenario):
        runner.compare(b, runner.ScenarioEval("x", "g", 1, 1.0, 1.0, True))
    with pytest.raises(ValueError):
        runner.compare(runner.ScenarioEval("x", "f", 0, 1.0, 1.0, True), c)
