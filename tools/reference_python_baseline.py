"""SURVEY §8(d) CPU baseline items (i)-(iii): the reference's OWN Python
planners, timed on this container's host (the reference cannot travel to the
GPU box, so this is measured here and committed under profiles/).

  (i)   single process: per-window ms and semantic candidates/s of
        brute_force_autoscale (cfg1 grid, 12^6 candidates), model_level_autoscale
        and greedy_autoscale (cfg2 70B windows)
  (ii)  the same fanned over windows with ProcessPoolExecutor(cpu_count)
  (iii) the literal per-candidate rate: _Evaluator.evaluate calls/s (6-op DAG)

    PYTHONDONTWRITEBYTECODE=1 python tools/reference_python_baseline.py
"""

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import opscaler as ref  # noqa: E402
from opscaler import autoscaler as A  # noqa: E402

from workloads import scenarios  # noqa: E402

A.MAX_ENUMERATION = 10**12


def _build(name):
    dag_spec, prof = scenarios.SCENARIOS[name]
    return ref.build_dag(dag_spec), ref.perfmodel.profiles_from_dict(prof)


def _points(name, k):
    tw = scenarios.trace_windows(name)
    n = len(tw["prefill_qps"])
    idx = [round(i * (n - 1) / max(1, k - 1)) for i in range(k)]
    return [(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i])) for i in idx if tw["prefill_qps"][i] > 0]


def job(args):
    mode, name, qps, L = args
    dag, prof = _build(name)
    pt = ref.WorkloadPoint(qps, L, "prefill")
    params = ref.AutoscaleParams(slo=scenarios.SLO[name]["prefill"])
    t = time.perf_counter()
    if mode == "oracle":
        A.brute_force_autoscale(dag, prof, pt, params, ref.BruteForceBounds(**scenarios.GRIDS[name]))
    elif mode == "model":
        A.model_level_autoscale(dag, prof, pt, params)
    else:
        A.greedy_autoscale(dag, prof, pt, params)
    return time.perf_counter() - t


def main():
    cores = os.cpu_count()
    res = {"host": {"cores": cores, "cpu": next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                                                 if l.startswith("model name")), "unknown")}}
    cases = [("oracle", "cfg1", 6, 12 ** 6), ("model", "cfg2", 12, None), ("operator", "cfg2", 12, None)]
    for mode, name, k, space in cases:
        jobs = [(mode, name, q, L) for q, L in _points(name, k)]
        single = [job(j) for j in jobs]
        t = time.perf_counter()
        with ProcessPoolExecutor(max_workers=cores) as ex:
            list(ex.map(job, jobs * max(1, cores // len(jobs))))
        pooled = time.perf_counter() - t
        n_pool = len(jobs) * max(1, cores // len(jobs))
        ms = sorted(x * 1e3 for x in single)
        r = {"windows": len(jobs), "median_ms": ms[len(ms) // 2], "max_ms": ms[-1],
             "pooled_windows_per_s": n_pool / pooled, "pooled_workers": cores}
        if space:
            r["semantic_candidates_per_s_single"] = space * len(single) / sum(single)
            r["semantic_candidates_per_s_pooled"] = space * n_pool / pooled
        res[f"{mode}/{name}"] = r
        print(mode, name, r, flush=True)
    # (iii) literal per-candidate rate of the reference evaluator (6-op chain)
    dag, prof = _build("cfg1")
    pt = ref.WorkloadPoint(10.0, 1024, "prefill")
    ev = A._Evaluator(dag, prof, pt, ref.AutoscaleParams(slo=0.5))
    cfgs = {op: A.OperatorConfig(p=1, r=2, b=1) for op in dag.node_ids}
    n, t = 0, time.perf_counter()
    while time.perf_counter() - t < 3.0:
        ev.evaluate(cfgs)
        n += 1
    res["evaluate_calls_per_s_per_core"] = n / (time.perf_counter() - t)
    print("evaluate/s", res["evaluate_calls_per_s_per_core"])
    os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
    with open(os.path.join(REPO, "profiles", "r01_reference_python_baseline.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
