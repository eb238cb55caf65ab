"""Pin the shared-placement restatement (oracle/opsc_oracle_place.c) to the
reference's own place() / request_energy / fill_device_energy outputs
(tests/golden/place.json, produced by tests/golden/make_golden_place.py)."""

import numpy as np
import pytest

import golden_cases as G
from paper_2511_02248_b200 import abi, model, placement, tables
from workloads import scenarios


def _setting_fleet(setting, slo, default_stream=False):
    name, n, caps, ccap, theta, expo, over = setting
    width = len(str(max(0, n - 1)))
    devs = [model.DeviceSpec(id=f"dev{i:0{width}d}", mem_cap=caps[i % len(caps)], compute_cap=ccap)
            for i in range(n)]
    return placement.SharedFleet(devs, slo, model.InterferenceParams(theta, expo), model.EnergyParams(),
                                 default_stream=default_stream, **over)


def _inputs(rec):
    src = G.load(rec["source"])
    c = next(c for c in src if c["name"] == rec["name"])
    prob = G.case_problem(c)
    params = G.case_params(c)
    win = G.case_windows(c)
    cfg = np.zeros((1, prob.n_ops, 3), np.int16)
    for op, p, r, b in rec["plan"]:
        cfg[0, prob.rank[op]] = (p, r, b)
    order = 0 if rec["source"] == "oracle.json" else 1
    return prob, params, win, cfg, order


def check_place(place_fn, rec, settings, variant="settings"):
    """variant: "settings" = shared placement, "default_stream" = no sharing."""
    prob, params, win, cfg, order = _inputs(rec)
    errs = []
    for s in settings:
        exp = rec[variant][s[0]]
        fleet = _setting_fleet(s, params.slo, default_stream=variant == "default_stream")
        out = place_fn(prob, win, cfg, np.ones(1, np.uint8), fleet, order)
        if "error" in exp:
            want = {"FleetExhausted": abi.W_FLEET_EXHAUSTED,
                    "InfeasiblePlacement": abi.W_INFEASIBLE_PLACEMENT}[exp["error"]]
            if not out.status[0] & want:
                errs.append((s[0], "status", int(out.status[0]), exp["error"]))
            continue
        na = int(out.n_assign[0])
        got_a = [[prob.ids[out.a_op[0, i]], int(out.a_replica[0, i]),
                  fleet.devices[out.a_device[0, i]].id, int(out.a_share[0, i]),
                  float(out.a_latency[0, i]).hex()] for i in range(na)]
        if got_a != exp["assignments"]:
            errs.append((s[0], "assignments", got_a[:4], exp["assignments"][:4]))
        got_d = [[fleet.devices[d].id, float(out.d_mem[0, d]).hex(), float(out.d_sm[0, d]).hex(),
                  float(out.d_energy[0, d]).hex()] for d in range(int(out.devices_used[0]))]
        if got_d != exp["devices"]:
            errs.append((s[0], "devices", got_d[:3], exp["devices"][:3]))
        for k in ("devices_used", "feasible"):
            if int(getattr(out, k)[0]) != int(exp[k]):
                errs.append((s[0], k, int(getattr(out, k)[0]), exp[k]))
        for k, ek in (("latency", "recomputed_latency"), ("energy", "energy"), ("memory", "memory")):
            if float(getattr(out, k)[0]).hex() != exp[ek]:
                errs.append((s[0], k, float(getattr(out, k)[0]).hex(), exp[ek]))
    return errs


CASES = G.load("place.json")["cases"]
SETTINGS = G.load("place.json")["settings"]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_oracle_place_shared(orc, idx):
    errs = check_place(orc.place_shared, CASES[idx], SETTINGS)
    assert not errs, (CASES[idx]["name"], errs[:3])


@pytest.mark.parametrize("idx", range(0, len(CASES)))
def test_oracle_default_stream(orc, idx):
    errs = check_place(orc.place_shared, CASES[idx], SETTINGS, "default_stream")
    assert not errs, (CASES[idx]["name"], errs[:3])
