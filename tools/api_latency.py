"""Per-point latency of the reference-shaped public API (dev tool, GPU):
planners.{brute_force,model_level,greedy}_autoscale on cfg2 windows, host
buffers in / ScalingPlan out, wall clock per call (Python packing included).

    python tools/api_latency.py [n_points]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import model, planners  # noqa: E402
from workloads import scenarios  # noqa: E402
from paper_2511_02248_b200.errors import NoStableConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dag, prof = scenarios.scenario("cfg2")
tw = scenarios.trace_windows("cfg2")
params = model.AutoscaleParams(slo=scenarios.SLO["cfg2"]["prefill"])
bounds = model.BruteForceBounds(**scenarios.GRIDS["cfg2"])
pts = [model.WorkloadPoint(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill") for i in range(n)]
for name, fn in (("brute_force", lambda p: planners.brute_force_autoscale(dag, prof, p, params, bounds, guards=False)),
                 ("model_level", lambda p: planners.model_level_autoscale(dag, prof, p, params)),
                 ("greedy", lambda p: planners.greedy_autoscale(dag, prof, p, params))):
    ts, raised = [], 0
    for p in pts[:3]:  # warm-up (library load, context, tables)
        try:
            fn(p)
        except NoStableConfig:
            pass
    for p in pts:
        t = time.perf_counter()
        try:
            fn(p)
        except NoStableConfig:  # the reference raises for these windows too (timed all the same)
            raised += 1
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{name}: median {statistics.median(ts):.3f} ms, max {max(ts):.3f} ms per point "
          f"({len(ts)} points, {raised} NoStableConfig)")
