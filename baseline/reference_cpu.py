"""The reference's OWN Python planners on this host's CPU cores.

BENCH INFRASTRUCTURE (bench.py's `--impl reference` arm and cpu_baseline
leg; tools/reference_python_baseline.py). The unmodified reference package is
imported from `baseline/_ref` (installed with `pip install --no-deps --target
baseline/_ref`, git-ignored, travels to the GPU box) or, in the build
container, from /root/reference/pkg/src. Nothing in the product package
imports it.

What runs is the reference's public planner API exactly as its CLI would call
it (`autoscaler.brute_force_autoscale` / `model_level_autoscale` /
`greedy_autoscale`, autoscaler.py:706, :596, :334). The one change is the
module global `autoscaler.MAX_ENUMERATION` (autoscaler.py:703, read at call
time :735), raised so brute force accepts the bench's 1.9e8-candidate
windows; its branch-and-bound with the greedy warm start (:767-826) then
runs as shipped. "All cores" = one worker process per host CPU
(ProcessPoolExecutor): the reference is GIL-bound, so its own
runner.sweep threads (runner.py:237-240) would not scale.
"""

from __future__ import annotations

import os
import statistics
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
PATHS = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def path():
    for p in PATHS:
        if os.path.isfile(os.path.join(p, "opscaler", "__init__.py")):
            return p
    return None


def available():
    return path() is not None


_W = {}  # per-process state: reference module + built scenario


def _init(ref_path, scenario, grid):
    if ref_path not in sys.path:
        sys.path.insert(0, ref_path)
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    import opscaler
    from opscaler import autoscaler
    from workloads import scenarios
    autoscaler.MAX_ENUMERATION = 10**15
    dag_spec, prof = scenarios.SCENARIOS[scenario]
    _W.update(ref=opscaler, A=autoscaler, dag=opscaler.build_dag(dag_spec),
              prof=opscaler.perfmodel.profiles_from_dict(prof),
              bounds=opscaler.BruteForceBounds(**grid) if grid else None)


def _plan(job):
    """One planner call; returns (seconds, decision summary)."""
    mode, qps, seq_len, phase, slo = job
    R, A = _W["ref"], _W["A"]
    pt = R.WorkloadPoint(qps, seq_len, phase)
    params = R.AutoscaleParams(slo=slo)
    t = time.perf_counter()
    try:
        if mode == "oracle":
            plan = A.brute_force_autoscale(_W["dag"], _W["prof"], pt, params, _W["bounds"])
        elif mode == "model":
            plan = A.model_level_autoscale(_W["dag"], _W["prof"], pt, params)
        else:
            plan = A.greedy_autoscale(_W["dag"], _W["prof"], pt, params)
        dt = time.perf_counter() - t
        out = (tuple(sorted((op, c.p, c.r, c.b) for op, c in plan.configs.items())),
               plan.objective, plan.feasible, plan.iteration_latency.hex())
    except R.OpscalerError as exc:
        dt = time.perf_counter() - t
        out = type(exc).__name__
    return dt, out


class Pool:
    """Worker processes with the reference imported and the scenario built."""

    def __init__(self, scenario, grid=None, workers=None):
        self.workers = workers or os.cpu_count() or 1
        self.ex = ProcessPoolExecutor(max_workers=self.workers, initializer=_init,
                                      initargs=(path(), scenario, grid))

    def run(self, jobs):
        """(wall seconds, [(seconds, decision)]) for all jobs over the pool."""
        t = time.perf_counter()
        res = list(self.ex.map(_plan, jobs, chunksize=max(1, len(jobs) // (4 * self.workers))))
        return time.perf_counter() - t, res

    def close(self):
        self.ex.shutdown()


def single(scenario, grid, jobs):
    """The same planner calls in THIS process (one core): per-window seconds."""
    _init(path(), scenario, grid)
    return [_plan(j) for j in jobs]


def per_window_stats(res, space=None):
    ms = sorted(dt * 1e3 for dt, _ in res)
    out = {"windows": len(ms), "median_ms": statistics.median(ms),
           "p99_ms": ms[min(len(ms) - 1, int(0.99 * len(ms)))], "max_ms": ms[-1]}
    if space:
        out["semantic_candidates_per_s"] = space * len(ms) / (sum(ms) * 1e-3)
    return out
