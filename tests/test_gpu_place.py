"""GPU shared placement (csrc/k_place.cu) against the reference's own
place()/energy outputs (golden) and the CPU oracle on large plans."""

import numpy as np
import pytest

import golden_cases as G
import test_oracle_place as TP
from paper_2511_02248_b200 import abi, model, placement, scenarios, tables

pytestmark = pytest.mark.gpu


def test_gpu_place_golden():
    errs = []
    for rec in TP.CASES:
        e = TP.check_place(placement.place_windows, rec, TP.SETTINGS)
        if e:
            errs.append((rec["name"], e[:2]))
    assert not errs, errs[:3]


def test_gpu_place_vs_oracle_large_plans(orc):
    """Model-level and greedy plans of the 70B trace (tens of replicas per op)."""
    from paper_2511_02248_b200 import _native
    prob = tables.pack_problem(*scenarios.scenario("cfg2"))
    tw = scenarios.trace_windows("cfg2")
    win = tables.window_arrays(tw["prefill_qps"][:24], tw["prefill_len"][:24], 0, 2.0)
    for mode in (abi.MODE_MODEL, abi.MODE_OPERATOR):
        prm = model.AutoscaleParams(slo=2.0)
        dec = _native.plan_windows_host(mode, prob, win, model=tables.pack_model(prob, prm),
                                        greedy=tables.pack_greedy(prob, prm))
        for theta, caps in ((0.5, [80e9]), (1.5, [180e9, 40e9])):
            devs = [model.DeviceSpec(id=f"g{i:04d}", mem_cap=caps[i % len(caps)]) for i in range(2048)]
            fleet = placement.SharedFleet(devs, 2.0, model.InterferenceParams(theta, 1.0), model.EnergyParams())
            gpu = placement.place_windows(prob, win, dec.cfg, dec.feasible, fleet, 1)
            cpu = orc.place_shared(prob, win, dec.cfg, dec.feasible, fleet, 1)
            for f in placement.PlacementArrays.FIELDS:
                assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (mode, theta, f)
