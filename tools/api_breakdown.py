"""Where the per-point API time goes (dev tool, GPU): for cfg2 (70B) prefill
windows, per call median of (a) the public planner call, (b) the bare C-ABI
host-buffer call with prepacked arguments, (c) its device span (first H2D ..
last D2H, CUDA events) -- (a)-(b) is Python, (b)-(c) launch/sync overhead.

    python tools/api_breakdown.py
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import _native, abi, model, planners, tables  # noqa: E402
from workloads import scenarios  # noqa: E402

dag, prof = scenarios.scenario("cfg2")
tw = scenarios.trace_windows("cfg2")
params = model.AutoscaleParams(slo=scenarios.SLO["cfg2"]["prefill"])
bounds = model.BruteForceBounds(**scenarios.GRIDS["cfg2"])
pts = [model.WorkloadPoint(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill") for i in range(60)]
prob = planners.packed_problem(dag, prof)
ctx = _native.context()
for name, mode, call in (
        ("brute_force", abi.MODE_ORACLE, lambda p: planners.brute_force_autoscale(dag, prof, p, params, bounds, guards=False)),
        ("model_level", abi.MODE_MODEL, lambda p: planners.model_level_autoscale(dag, prof, p, params)),
        ("greedy", abi.MODE_OPERATOR, lambda p: planners.greedy_autoscale(dag, prof, p, params))):
    kw = dict(grid=tables.pack_grid(prob, params, bounds), model=tables.pack_model(prob, params),
              greedy=tables.pack_greedy(prob, params))
    place = tables.pack_place()
    tcap = 4096 if mode == abi.MODE_OPERATOR else 0
    out = tables.DecisionArrays(1, prob.n_ops, tcap)
    a, b, c = [], [], []
    for rep in range(3):
        for p in pts:
            t = time.perf_counter()
            try:
                call(p)
            except Exception:
                pass
            a.append(time.perf_counter() - t)
            win = tables.pack_windows([p], params.slo, params.epsilon)
            t = time.perf_counter()
            ctx.plan_windows(mode, prob, win, place=place, out=out, trace_cap=tcap, **kw)
            b.append(time.perf_counter() - t)
            c.append(ctx.last_ms() * 1e-3)
    m = lambda x: statistics.median(x[60:]) * 1e3
    print(f"{name}: public API {m(a):.3f} ms | C-ABI call {m(b):.3f} ms | device span {m(c):.3f} ms")
