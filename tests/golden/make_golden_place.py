"""Freeze golden vectors of the reference's shared placement (Alg. 2).

Build container only (imports /root/reference). For decided plans of the
golden planner cases (tests/golden/{oracle,model,greedy}.json inputs) the
reference's own placement.place() (placement.py:399-462) and
default_stream_place() (:465-491) with their metrics
(request_energy, fill_device_energy, provisioned_memory; metrics.py:84-132)
are run on several fleets / interference settings; every float is stored as
float.hex().

    PYTHONHASHSEED=0 PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_place.py
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import opscaler as ref  # noqa: E402
from opscaler import autoscaler as A  # noqa: E402
from opscaler import metrics as M  # noqa: E402
from opscaler import placement as PL  # noqa: E402
from opscaler import perfmodel as PM  # noqa: E402

import make_golden as MG  # noqa: E402

A.MAX_ENUMERATION = 10**12
H = MG.H

SETTINGS = [
    # (name, n_devices, mem_caps, compute_cap, theta, exponent, place-param overrides)
    ("b200", 512, [180e9], 1.0, 0.5, 1.0, {}),
    ("a100", 512, [80e9], 1.0, 0.5, 1.0, {}),
    ("hetero", 512, [80e9, 40e9, 180e9, 96e9], 1.0, 0.5, 1.0, {}),
    ("theta0", 512, [80e9], 1.0, 0.0, 1.0, {}),
    ("strong", 512, [80e9], 1.0, 1.5, 1.0, {"max_sm_load": 2.5}),
    ("weights", 512, [120e9], 1.2, 0.8, 1.0, {"slack_weight_mem": 0.9, "slack_weight_compute": 0.1}),
    ("small", 6, [80e9], 1.0, 0.5, 1.0, {}),
    ("tiny_mem", 64, [3.0e8], 1.0, 0.5, 1.0, {}),
]


def fleet(n, caps, ccap):
    width = len(str(max(0, n - 1)))
    # ids deliberately not in creation order: placement sorts by id
    ids = [f"dev{i:0{width}d}" for i in range(n)]
    rng = np.random.default_rng(n)
    order = rng.permutation(n)
    return [PL.DeviceSpec(id=ids[i], mem_cap=caps[i % len(caps)], compute_cap=ccap) for i in order]


def place_json(plan, dag, profiles, point, setting, place_fn=PL.place):
    name, n, caps, ccap, theta, expo, over = setting
    prof = PM.ProfileSet(profiles.profiles, profiles.link_bandwidth,
                         PM.InterferenceParams(theta=theta, exponent=expo))
    fl = fleet(n, caps, ccap)
    pp = PL.PlacementParams(slo=plan_slo[0], **over)
    try:
        placed = place_fn(plan, dag, prof, fl, pp, point)
    except ref.OpscalerError as exc:
        return {"error": type(exc).__name__}
    ep = M.EnergyParams()
    energy = M.request_energy(plan, placed, dag, prof, point, ep)
    M.fill_device_energy(placed, plan, dag, prof, point, ep)
    return {
        "assignments": [[a.op_id, a.replica_index, a.device_id, a.sm_share,
                         H(a.interference_adjusted_latency)] for a in placed.assignments],
        "devices": [[d, H(l.mem_used), H(l.sm_demand), H(l.energy)]
                    for d, l in placed.device_loads.items()],
        "devices_used": placed.devices_used,
        "feasible": placed.feasible,
        "recomputed_latency": H(placed.recomputed_latency),
        "energy": H(energy),
        "memory": H(M.provisioned_memory(plan, placed)),
    }


plan_slo = [0.0]


def main():
    out = []
    for src, runner_fn in (("oracle.json", "oracle"), ("model.json", "model"), ("greedy.json", "greedy")):
        cases = json.load(open(os.path.join(HERE, src)))
        for c in cases[::3] if src != "greedy.json" else cases[::2]:
            if "error" in c["expected"] or not c["expected"]["feasible"]:
                continue
            dag_spec, prof_d = (MG.S.SCENARIOS[c["scenario"]] if "scenario" in c
                                else (c["dag"], c["profiles"]))
            dag, profiles = MG.build(dag_spec, prof_d)
            p = c["point"]
            pt = ref.WorkloadPoint(float.fromhex(p["qps"]), p["seq_len"], p["phase"])
            pr = c["params"]
            params = ref.AutoscaleParams(
                slo=float.fromhex(pr["slo"]), epsilon=float.fromhex(pr["epsilon"]),
                b_max=pr["b_max"], parallelism=tuple(pr["parallelism"]), r_cap=pr["r_cap"],
                max_iterations=pr.get("max_iterations", 10_000),
                prune_excess_replicas=pr.get("prune_excess_replicas", False))
            if runner_fn == "oracle":
                b = c["bounds"]
                plan = A.brute_force_autoscale(dag, profiles, pt, params, ref.BruteForceBounds(
                    r_max=b["r_max"], b_max=b["b_max"], parallelism=tuple(b["parallelism"])))
            elif runner_fn == "model":
                plan = A.model_level_autoscale(dag, profiles, pt, params)
            else:
                plan = A.greedy_autoscale(dag, profiles, pt, params)
            if sum(cf.r for cf in plan.configs.values()) > 300:
                continue  # keep the fixture small; large plans are covered GPU-vs-oracle
            plan_slo[0] = params.slo
            rec = {"source": src, "name": c["name"],
                   "plan": [[op, cf.p, cf.r, cf.b] for op, cf in plan.configs.items()],
                   "settings": {}}
            for s in SETTINGS:
                rec["settings"][s[0]] = place_json(plan, dag, profiles, pt, s)
            # the no-sharing variant (placement.py:465-491) on the same fleets
            rec["default_stream"] = {s[0]: place_json(plan, dag, profiles, pt, s, PL.default_stream_place)
                                     for s in SETTINGS}
            out.append(rec)
    json.dump({"settings": [[s[0], s[1], s[2], s[3], s[4], s[5], s[6]] for s in SETTINGS],
               "cases": out}, open(os.path.join(HERE, "place.json"), "w"), separators=(",", ":"))
    n_err = sum(1 for r in out for v in r["settings"].values() if "error" in v)
    n_inf = sum(1 for r in out for v in r["settings"].values() if "error" not in v and not v["feasible"])
    n_asg = sum(len(v.get("assignments", [])) for r in out for v in r["settings"].values())
    print(f"place: {len(out)} plans x {len(SETTINGS)} settings, {n_err} errors, "
          f"{n_inf} infeasible placements, {n_asg} assignments")


if __name__ == "__main__":
    main()
