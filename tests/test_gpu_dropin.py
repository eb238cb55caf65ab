"""The drop-in seam on the B200, with the UNMODIFIED reference package.

`install(opscaler)` rebinds the reference's planners, placement, runner.sweep
and cli.cmd_autoscale (installer.py). Here the reference itself is imported
(tests/refpkg.py: baseline/_ref on the GPU box) and driven through its own
entry points -- runner.plan_for_mode (runner.py:38-52), runner.run_point
(runner.py:55-105) and cli.main (cli.py:299-313) -- and every result is
compared with what the same reference functions return WITHOUT the drop-in,
run live on this box's CPU: same classes, same reprs (float repr is exact),
same exceptions, byte-identical CLI artefacts.
"""

import contextlib
import hashlib
import io
import os
import tempfile

import pytest

import golden_cases as G
import refpkg
from workloads import scenarios

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    op = refpkg.import_reference()
    import importlib
    for sub in ("runner", "cli"):
        importlib.import_module("opscaler." + sub)
    from paper_2511_02248_b200 import _native
    _native.load()
    assert _native.device_count() >= 1, "no CUDA device"
    return op


@contextlib.contextmanager
def installed(op):
    from paper_2511_02248_b200 import install
    undo = install(op)
    try:
        yield
    finally:
        undo()


def _build(op, cfg):
    dag_spec, prof = scenarios.SCENARIOS[cfg]
    return op.build_dag(dag_spec), op.perfmodel.profiles_from_dict(prof)


def _points(op, cfg, windows):
    tw = scenarios.trace_windows(cfg)
    out = []
    for w in windows:
        for ph in ("prefill", "decode"):
            q = float(tw[ph + "_qps"][w])
            if q > 0:
                out.append(op.WorkloadPoint(q, int(tw[ph + "_len"][w]), ph))
    return out


def _cases(op):
    """(mode, cfg, point, params, bounds) spanning all three modes, three DAGs,
    epsilon headroom, prune, infeasible SLOs and NoStableConfig."""
    A = op.autoscaler
    cs = []
    g1 = op.BruteForceBounds(**{k: v for k, v in scenarios.GRIDS["cfg1"].items()})
    g3 = op.BruteForceBounds(**{k: v for k, v in scenarios.GRIDS["cfg3s"].items()})
    for pt in _points(op, "cfg1", [0]):
        slo = scenarios.SLO["cfg1"][pt.phase]
        for mode in ("oracle", "model", "operator"):
            cs.append((mode, "cfg1", pt, A.AutoscaleParams(slo=slo), g1))
            cs.append((mode, "cfg1", pt, A.AutoscaleParams(slo=slo, epsilon=0.1 * slo), g1))
        cs.append(("oracle", "cfg1", pt, A.AutoscaleParams(slo=1e-5), g1))      # infeasible SLO
    for pt in _points(op, "cfg3s", [0, 17]):
        cs.append(("oracle", "cfg3s", pt, A.AutoscaleParams(slo=scenarios.SLO["cfg3s"][pt.phase]), g3))
    for pt in _points(op, "cfg2", [0, 13, 40]):
        slo = scenarios.SLO["cfg2"][pt.phase]
        cs.append(("model", "cfg2", pt, A.AutoscaleParams(slo=slo), None))
        cs.append(("operator", "cfg2", pt, A.AutoscaleParams(slo=slo, prune_excess_replicas=True), None))
    for pt in _points(op, "cfg3", [5]):
        slo = scenarios.SLO["cfg3"][pt.phase]
        cs.append(("operator", "cfg3", pt, A.AutoscaleParams(slo=slo, epsilon=0.05 * slo), None))
        cs.append(("model", "cfg3", pt, A.AutoscaleParams(slo=slo), None))
    hot = op.WorkloadPoint(1e9, 2048, "prefill")                                 # NoStableConfig
    for mode in ("oracle", "model", "operator"):
        cs.append((mode, "cfg1", hot, A.AutoscaleParams(slo=0.5), g1))
    # the reference's own guard: 10 operators refused by brute force
    cs.append(("oracle", "cfg2", _points(op, "cfg2", [0])[0], A.AutoscaleParams(slo=2.0),
               op.BruteForceBounds(r_max=1, b_max=1)))
    return cs


def _outcome(fn):
    try:
        return "ok", fn()
    except Exception as exc:  # the reference's own exception classes
        return "raise", exc


def _same_exc(a, b):
    return type(a) is type(b) and str(a) == str(b)


def test_plan_for_mode_matches_live_reference(ref):
    """runner.plan_for_mode in all three modes: the drop-in returns the
    reference's own ScalingPlan / OperatorConfig / PredictedSojourn objects
    whose repr (exact floats, move trace included) equals the reference's."""
    R = ref.runner
    cases = _cases(ref)
    built = {cfg: _build(ref, cfg) for cfg in {c[1] for c in cases}}
    want = [_outcome(lambda c=c: R.plan_for_mode(c[0], *built[c[1]], c[2], c[3], c[4])) for c in cases]
    with installed(ref):
        assert hasattr(ref.autoscaler.greedy_autoscale, "__wrapped__")  # the drop-in wrapper
        got = [_outcome(lambda c=c: R.plan_for_mode(c[0], *built[c[1]], c[2], c[3], c[4])) for c in cases]
    n_plans = 0
    for c, (wk, w), (gk, g) in zip(cases, want, got):
        assert wk == gk, (c[0], c[1], c[2], w, g)
        if wk == "raise":
            assert _same_exc(w, g), (c[0], c[1], w, g)
            continue
        n_plans += 1
        assert type(g) is ref.autoscaler.ScalingPlan
        assert all(type(v) is ref.autoscaler.OperatorConfig for v in g.configs.values())
        assert all(type(v) is ref.autoscaler.PredictedSojourn for v in g.predicted.values())
        assert repr(g) == repr(w), (c[0], c[1], c[2])
    kinds = {(c[0], w[0]) for c, w in zip(cases, want)}
    assert {("oracle", "ok"), ("model", "ok"), ("operator", "ok"), ("oracle", "raise"),
            ("model", "raise"), ("operator", "raise")} <= kinds
    assert n_plans >= 25


@pytest.mark.parametrize("placement_mode", ["shared", "default_stream"])
def test_run_point_matches_live_reference(ref, placement_mode):
    """runner.run_point: plan -> (rerouted) placement -> the reference's own
    metrics; PointResult reprs (plan, Placement, ScenarioEval) identical."""
    R = ref.runner
    A = ref.autoscaler
    fleet = ref.make_fleet(64)
    cases = [c for c in _cases(ref) if not (c[1] == "cfg2" and c[0] == "oracle")]
    built = {cfg: _build(ref, cfg) for cfg in {c[1] for c in cases}}

    def run(c):
        return R.run_point(c[0], *built[c[1]], fleet, c[2], c[3], placement_mode, None, c[4])

    want = [_outcome(lambda c=c: run(c)) for c in cases]
    with installed(ref):
        got = [_outcome(lambda c=c: run(c)) for c in cases]
    placed = 0
    for c, (wk, w), (gk, g) in zip(cases, want, got):
        assert wk == gk, (c[0], c[1], w, g)
        if wk == "raise":
            assert _same_exc(w, g), (c[0], c[1], w, g)
            continue
        assert type(g) is R.PointResult
        assert repr(g.plan) == repr(w.plan)
        assert repr(g.placement) == repr(w.placement), (c[0], c[1], c[2])
        assert repr(g.evaluation) == repr(w.evaluation)
        placed += g.placement is not None
    assert placed >= 10
    assert not hasattr(A.brute_force_autoscale, "__wrapped__")  # uninstalled again


CLI_IN = os.path.join(os.path.dirname(__file__), "golden", "cli")


def _run_cli(main, argv):
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "out")
        err = io.StringIO()
        cwd = os.getcwd()
        os.chdir(CLI_IN)
        try:
            with contextlib.redirect_stderr(err):
                rc = main(argv + ["--out", out])
        finally:
            os.chdir(cwd)
        files = {}
        if os.path.isdir(out):
            for name in sorted(os.listdir(out)):
                with open(os.path.join(out, name), "rb") as fh:
                    files[name] = hashlib.sha256(fh.read()).hexdigest()
        return rc, err.getvalue(), files


def test_reference_cli_main_on_the_gpu(ref):
    """The reference's own `opscaler autoscale | sweep` (cli.main) with the
    drop-in installed: every artefact of the 22 golden CLI cases (frozen from
    the reference CLI) byte-identical, same exit codes and stderr."""
    cases = G.load("cli.json")
    with installed(ref):
        assert hasattr(ref.cli.cmd_autoscale, "__wrapped__")
        for c in cases:
            rc, err, files = _run_cli(ref.cli.main, c["argv"])
            assert files == c["files"], c["name"]
            assert rc == c["exit"], c["name"]
            assert err == c["stderr"], c["name"]
