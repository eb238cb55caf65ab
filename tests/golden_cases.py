"""Load the golden fixtures (tests/golden/*.json, produced by running the
reference itself via tests/golden/make_golden.py) into packed inputs."""

import functools
import json
import os

import numpy as np

from paper_2511_02248_b200 import model, tables
from workloads import scenarios

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def F(h):
    return float.fromhex(h)


def case_problem(c):
    if "scenario" in c:
        dag, prof = scenarios.SCENARIOS[c["scenario"]]
    else:
        dag, prof = c["dag"], c["profiles"]
    return tables.pack_problem(model.build_dag(dag), model.profiles_from_dict(prof))


def case_params(c):
    p = c["params"]
    par = p["parallelism"]
    par = {k: tuple(v) for k, v in par.items()} if isinstance(par, dict) else tuple(par)
    return model.AutoscaleParams(slo=F(p["slo"]), epsilon=F(p["epsilon"]), b_max=p["b_max"],
                                 parallelism=par, r_cap=p["r_cap"],
                                 max_iterations=p.get("max_iterations", 10_000),
                                 prune_excess_replicas=p.get("prune_excess_replicas", False))


def case_bounds(c):
    b = c["bounds"]
    return model.BruteForceBounds(r_max=b["r_max"], b_max=b["b_max"],
                                  parallelism=None if b["parallelism"] is None else tuple(b["parallelism"]))


def case_point(c):
    pt = c["point"]
    return model.WorkloadPoint(F(pt["qps"]), pt["seq_len"], pt["phase"])


def case_windows(c):
    params = case_params(c)
    return tables.pack_windows([case_point(c)], params.slo, params.epsilon)


def fleet_for(kind):
    if kind == "metrics":
        return model.make_fleet(256, mem_cap=180e9)
    if kind == "metrics_small_fleet":
        return model.make_fleet(4, mem_cap=40e9)
    if kind == "metrics_tiny_cap":
        return model.make_fleet(64, mem_cap=2.0e8)
    if kind == "model_metrics":
        return model.make_fleet(4096, mem_cap=180e9)
    raise KeyError(kind)


def compare_plan(plan, exp, problem):
    """Bit-exact comparison of a materialised plan against a golden plan."""
    errs = []
    got_cfg = [[op, c.p, c.r, c.b] for op, c in plan.configs.items()]
    if got_cfg != exp["configs"]:
        errs.append(f"configs {got_cfg} != {exp['configs']}")
    if plan.objective != exp["objective"]:
        errs.append(f"objective {plan.objective} != {exp['objective']}")
    if plan.feasible != exp["feasible"]:
        errs.append(f"feasible {plan.feasible} != {exp['feasible']}")
    if plan.iteration_latency.hex() != exp["iteration_latency"]:
        errs.append(f"latency {plan.iteration_latency.hex()} != {exp['iteration_latency']}")
    if plan.critical_path != exp["critical_path"]:
        errs.append(f"path {plan.critical_path} != {exp['critical_path']}")
    if "trace" in exp:
        got_tr = []
        for t in plan.trace:
            e = {"action": t["action"], "objective": t["objective"]}
            if "op" in t:
                e["op"] = t["op"]
                e["to"] = [t["to"]["R"], t["to"]["B"], t["to"]["P"]]
                e["latency"] = t["latency"].hex()
            got_tr.append(e)
        if got_tr != exp["trace"]:
            errs.append(f"trace {got_tr} != {exp['trace']}")
    for op, fields in exp["predicted"].items():
        p = plan.predicted[op]
        got = [p.op_latency.hex(), p.lam.hex(), p.mu.hex(), p.utilization.hex(),
               p.wait.hex(), p.service.hex(), p.comm.hex(), p.stable]
        if got != fields:
            errs.append(f"predicted[{op}] {got} != {fields}")
    return errs


def compare_metrics(m, exp):
    if exp is None:
        return [] if m is None else [f"unexpected metrics {m}"]
    if "error" in exp:
        return [] if (m is not None and m.error == exp["error"]) else [f"metrics {m} != {exp}"]
    errs = []
    if m is None or m.error:
        return [f"metrics {m} != {exp}"]
    if m.devices_used != exp["devices"]:
        errs.append(f"devices {m.devices_used} != {exp['devices']}")
    if m.energy_joules.hex() != exp["energy"]:
        errs.append(f"energy {m.energy_joules.hex()} != {exp['energy']}")
    if m.memory_bytes.hex() != exp["memory"]:
        errs.append(f"memory {m.memory_bytes.hex()} != {exp['memory']}")
    return errs
