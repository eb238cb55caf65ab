"""Throughput under a fixed GPU budget.

The reference has no such operation; SURVEY §8(d) proposes it as an
extension: per window, the largest arrival rate whose min-objective feasible
decision fits an N-device fleet (default-stream placement `devices_used <=
N`, placement.py:465-491), found by bisection over the rate with the same
planning kernels. Parity is therefore UNPINNED against the reference; the
GPU search is checked bit-for-bit against the same search driven by the CPU
oracle (tests/test_gpu_capacity.py).

Search (batched k-ary bisection): each round evaluates `fan` rates for every
window in ONE planning launch set (W x fan windows: menus / compose / decode
/ materialise, or the model-level / greedy planners), keeps the largest
rate that fits as the new lower bound and the next larger rate that does
not as the upper bound. Round 0 is geometric (2^-fan/2 .. 2^fan/2 times the
window's rate); later rounds are linear inside [lo, hi). With fan = 32 each
round narrows the bracket 33x.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, abi, model, tables

_MODES = {"oracle": abi.MODE_ORACLE, "model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR}
# any of these makes a rate "not fit": no feasible decision, planner errors,
# or a default-stream placement beyond the fleet
_FAIL = (abi.W_FLEET_EXHAUSTED | abi.W_INFEASIBLE_PLACEMENT | abi.W_NO_STABLE_PARAMS | abi.W_NO_STABLE_BOUNDS
         | abi.W_NO_STABLE_MODEL | abi.W_NO_STABLE_INIT | abi.W_UNSTABLE_ROUNDING | abi.W_ZERO_DIVISION)


def fits(arrays, budget):
    return ((arrays.feasible == 1) & ((arrays.status & _FAIL) == 0) & (arrays.devices <= budget))


@dataclass
class CapacityResult:
    qps: np.ndarray        # [W] largest fitting rate found (0.0: none fits)
    upper: np.ndarray      # [W] smallest non-fitting rate above it (inf: none found)
    cfg: np.ndarray        # [W, n, 3] decision at `qps`
    devices: np.ndarray    # [W] default-stream devices of that decision
    objective: np.ndarray  # [W]
    latency: np.ndarray    # [W]
    rounds: int
    evaluated: int         # planning problems solved (windows x rates)


def device_evaluator(mode, problem, grid=None, model_spec=None, greedy=None, place=None):
    m = _MODES[mode] if isinstance(mode, str) else mode

    def evaluate(win: tables.WindowArrays):
        return _native.plan_windows_host(m, problem, win, grid=grid, model=model_spec, place=place,
                                         greedy=greedy, trace_cap=0)
    return evaluate


def max_qps_under_budget(dag, profiles, points, params, mode="oracle", bounds=None, budget=8,
                         mem_cap=80e9, fan=32, rel_tol=1e-6, max_rounds=16, evaluate=None):
    """Per point: the largest qps (same seq_len / phase / SLO) whose decision
    is SLO-feasible and fits `budget` devices of `mem_cap` bytes."""
    problem = tables.pack_problem(dag, profiles)
    for ph in sorted({p.phase for p in points}):
        problem.require_phase(ph)
    m = _MODES[mode] if isinstance(mode, str) else mode
    if m == abi.MODE_ORACLE and bounds is None:
        bounds = model.BruteForceBounds()
    place = tables.pack_place(model.make_fleet(budget, mem_cap))
    if evaluate is None:
        evaluate = device_evaluator(
            m, problem, grid=tables.pack_grid(problem, params, bounds) if m == abi.MODE_ORACLE else None,
            model_spec=tables.pack_model(problem, params),
            greedy=tables.pack_greedy(problem, params) if m == abi.MODE_OPERATOR else None, place=place)
    return search(points, params, evaluate, problem.n_ops, budget, fan, rel_tol, max_rounds)


def search(points, params, evaluate, n_ops, budget, fan=32, rel_tol=1e-6, max_rounds=16):
    """The k-ary bisection over `evaluate(WindowArrays) -> DecisionArrays`
    (GPU planners in the product; the CPU oracle in the parity tests)."""
    W, K = len(points), int(fan)
    base = np.array([p.qps if p.qps > 0 else 1.0 for p in points], dtype=np.float64)
    seq = np.array([p.seq_len for p in points], dtype=np.int32)
    ph = np.array([tables.PHASE_INDEX[p.phase] for p in points], dtype=np.uint8)
    lo = np.zeros(W)
    hi = np.full(W, np.inf)
    best = {"cfg": np.zeros((W, n_ops, 3), np.int16), "devices": np.zeros(W, np.int32),
            "objective": np.zeros(W, np.int32), "latency": np.zeros(W)}
    evaluated = 0
    rounds = 0
    active = np.ones(W, dtype=bool)
    geo = np.exp2(np.arange(K, dtype=np.float64) - K // 2)
    frac = np.arange(1, K + 1, dtype=np.float64) / (K + 1)
    for rounds in range(1, max_rounds + 1):
        idx = np.nonzero(active)[0]
        if not idx.size:
            break
        if rounds == 1:
            grid = base[idx, None] * geo[None, :]
        else:
            l, h = lo[idx], hi[idx]
            unb = ~np.isfinite(h)
            grid = np.empty((idx.size, K))
            # unbounded above: keep doubling from lo; bracketed: linear inside
            grid[unb] = l[unb, None] * np.exp2(np.arange(1, K + 1, dtype=np.float64))[None, :]
            grid[~unb] = l[~unb, None] + (h[~unb] - l[~unb])[:, None] * frac[None, :]
        A = idx.size
        win = tables.WindowArrays(
            qps=np.ascontiguousarray(grid.reshape(-1)), seq_len=np.repeat(seq[idx], K),
            phase=np.repeat(ph[idx], K), slo=np.full(A * K, float(params.slo)),
            eps=np.full(A * K, float(params.epsilon)))
        out = evaluate(win)
        evaluated += A * K
        ok = fits(out, budget).reshape(A, K)
        for a, w in enumerate(idx):
            good = np.nonzero(ok[a])[0]
            if good.size:
                k = int(good[-1])
                if grid[a, k] > lo[w]:
                    lo[w] = grid[a, k]
                    i = a * K + k
                    best["cfg"][w] = out.cfg[i]
                    best["devices"][w] = out.devices[i]
                    best["objective"][w] = out.objective[i]
                    best["latency"][w] = out.latency[i]
            above = np.nonzero(~ok[a] & (grid[a] > lo[w]))[0]
            if above.size:
                hi[w] = min(hi[w], float(grid[a, above[0]]))
            if rounds == 1 and not good.size:
                active[w] = False  # nothing fits even at 2^-fan/2 x the rate: capacity 0
            elif np.isfinite(hi[w]) and hi[w] - lo[w] <= rel_tol * lo[w]:
                active[w] = False
    return CapacityResult(qps=lo, upper=hi, cfg=best["cfg"], devices=best["devices"],
                          objective=best["objective"], latency=best["latency"], rounds=rounds,
                          evaluated=evaluated)
