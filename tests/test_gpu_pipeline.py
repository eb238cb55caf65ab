"""Trace -> decisions fully on the device (windowize + planners) equals the
host-side flow: reference-equivalent windowize, then the per-window planners."""

import numpy as np
import pytest

from paper_2511_02248_b200 import model, pipeline, planners, workload
from workloads import scenarios

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["operator", "model", "oracle"])
def test_trace_pipeline_matches_per_window_planners(mode):
    cfg = "cfg2" if mode != "oracle" else "cfg1"
    spec = scenarios.TRACES[cfg]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    if cfg == "cfg2":
        recs = [r for r in recs if r.arrival_time < 900.0]  # 15 windows
    dag, prof = scenarios.scenario(cfg)
    params = {ph: model.AutoscaleParams(slo=scenarios.SLO[cfg][ph]) for ph in ("prefill", "decode")}
    bounds = model.BruteForceBounds(**scenarios.GRIDS[cfg]) if mode == "oracle" else None
    tp = pipeline.TracePlanner(dag, prof, params, mode, bounds)
    arr = np.array([r.arrival_time for r in recs])
    li = np.array([r.input_len for r in recs])
    lo = np.array([r.output_len for r in recs])
    got = tp.plans(arr, li, lo)
    wins = workload.windowize(recs, spec["window_len"], spec["quantile"])
    assert len(got) == len(wins)
    for ph_i, ph in enumerate(("prefill", "decode")):
        pts = [w[ph_i] for w in wins]
        exp = planners.plan_windows(dag, prof, pts, params[ph], mode, bounds)
        for g, e in zip(got, exp):
            assert (g[ph_i] is None) == (e is None)
            if e is not None:
                assert g[ph_i].to_dict() == e.to_dict()
