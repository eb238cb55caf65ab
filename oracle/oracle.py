"""ctypes front-end of the CPU restatement (oracle/opsc_oracle.c).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module. The product
package never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_02248_b200 import abi, tables

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libopsc_oracle.so")

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        D, I, U = C.c_double, C.c_int32, C.c_uint32
        L.orc_op_latency.restype = D
        L.orc_op_latency.argtypes = [D, D, D, D, C.c_int64, C.c_int64, C.c_int64]
        L.orc_comm_time.restype = D
        L.orc_comm_time.argtypes = [D, D, C.c_int64, C.c_int64, D]
        L.orc_op_memory.restype = D
        L.orc_op_memory.argtypes = [D, D, D, C.c_int64, C.c_int64, C.c_int64]
        L.orc_erlang_c.restype = D
        L.orc_erlang_c.argtypes = [I, D]
        L.orc_expected_wait.restype = D
        L.orc_expected_wait.argtypes = [D, D, I]
        L.orc_strict_min_replicas.restype = I
        L.orc_strict_min_replicas.argtypes = [D, D, I]
        L.orc_py_sum.restype = D
        L.orc_py_sum.argtypes = [P, I]
        L.orc_critical_path.restype = D
        L.orc_critical_path.argtypes = [P, P, P]
        L.orc_predict.restype = I
        L.orc_predict.argtypes = [P, D, I, I, I, I, I, I, P, P]
        L.orc_menu_build.argtypes = [P, P, abi.OpscWindows, P, P, I]
        L.orc_stability_check.argtypes = [P, P, abi.OpscWindows, P, I]
        L.orc_compose_argmin.argtypes = [P, P, abi.OpscWindows, P, I, I, P, I]
        L.orc_menu_fallback.argtypes = [P, P, I, P, P]
        L.orc_decode_decisions.argtypes = [P, P, I, P, P, P, P, P]
        L.orc_model_grid.argtypes = [P, P, abi.OpscWindows, P, P, P, I]
        L.orc_materialize.argtypes = [P, abi.OpscWindows, I, P, abi.OpscDecisions, I]
        L.orc_plan_windows.argtypes = [I, P, P, P, P, P, abi.OpscWindows, abi.OpscDecisions, I]
        L.orc_greedy.argtypes = [P, P, abi.OpscWindows, P, P, P, abi.OpscDecisions, I]
        L.orc_place_shared.argtypes = [P, P, abi.OpscWindows, P, P, I, abi.OpscPlacement, I]
        L.orc_windowize.argtypes = [abi.OpscTraceRecords, D, D, I, P, P, P]
        L.orc_windowize.restype = I
        for f in ("orc_menu_build", "orc_stability_check", "orc_compose_argmin",
                  "orc_menu_fallback", "orc_decode_decisions", "orc_model_grid",
                  "orc_materialize", "orc_plan_windows", "orc_greedy", "orc_place_shared"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def threads():
    return int(os.environ.get("OPSC_ORACLE_THREADS", os.cpu_count() or 1))


def ref(x):
    return C.cast(C.byref(x), C.c_void_p)


def plan_windows(mode, problem, windows, grid=None, model=None, place=None, n_threads=None,
                 greedy=None, trace_cap=4096):
    """Whole pipeline (menus -> argmin -> decode -> materialise) on the CPU."""
    place = place or tables.pack_place()
    out = tables.DecisionArrays(windows.n, problem.n_ops,
                                trace_cap if mode == abi.MODE_OPERATOR else 0)
    g = grid if grid is not None else abi.OpscGrid()
    m = model if model is not None else abi.OpscModelSpec()
    gs = greedy if greedy is not None else abi.OpscGreedySpec()
    rc = lib().orc_plan_windows(mode, ref(problem.table), ref(g), ref(m), ref(gs), ref(place.spec),
                                windows.struct(), out.struct(), n_threads or threads())
    if rc != abi.OK:
        raise RuntimeError(f"oracle status {rc}")
    return out


def menus(problem, grid, windows, n_threads=None):
    E = grid.menu_off[problem.n_ops]
    mw = np.zeros((windows.n, E), dtype=np.float64)
    st = np.zeros(windows.n, dtype=np.uint32)
    lib().orc_menu_build(ref(problem.table), ref(grid), windows.struct(), mw.ctypes.data,
                         st.ctypes.data, n_threads or threads())
    return mw, st


def compose(problem, grid, windows, menu_w, shard=0, n_shards=1, n_threads=None, key=None):
    key = np.full(windows.n, abi.KEY_INFEASIBLE, dtype=np.int64) if key is None else key
    rc = lib().orc_compose_argmin(ref(problem.table), ref(grid), windows.struct(),
                                  np.ascontiguousarray(menu_w).ctypes.data, shard, n_shards,
                                  key.ctypes.data, n_threads or threads())
    if rc != abi.OK:
        raise RuntimeError(f"oracle status {rc}")
    return key


def windowize(arrival, input_len, output_len, window_len=60.0, quantile=0.95, max_windows=1 << 20):
    """(prefill_qps, prefill_len, decode_qps) per window, CPU restatement."""
    a = np.ascontiguousarray(arrival, dtype=np.float64)
    i = np.ascontiguousarray(input_len, dtype=np.int32)
    o = np.ascontiguousarray(output_len, dtype=np.int32)
    rec = abi.OpscTraceRecords(len(a), a.ctypes.data, i.ctypes.data, o.ctypes.data)
    pq = np.zeros(max_windows); pl = np.zeros(max_windows, dtype=np.int32); dq = np.zeros(max_windows)
    n = lib().orc_windowize(rec, window_len, quantile, max_windows, pq.ctypes.data, pl.ctypes.data,
                            dq.ctypes.data)
    if n < 0:
        raise ValueError("more windows than max_windows")
    return pq[:n].copy(), pl[:n].copy(), dq[:n].copy()


def place_shared(problem, windows, cfg, plan_feasible, fleet, config_order, n_threads=None):
    """Shared placement + metrics of decided plans on the CPU (PlacementArrays)."""
    from paper_2511_02248_b200 import placement
    cfg = np.ascontiguousarray(cfg, dtype=np.int16)
    feas = np.ascontiguousarray(plan_feasible, dtype=np.uint8)
    ca, cd = placement.capacities(cfg, fleet.spec.n_devices)
    out = placement.PlacementArrays(windows.n, ca, cd)
    rc = lib().orc_place_shared(ref(problem.table), ref(fleet.spec), windows.struct(), cfg.ctypes.data,
                                feas.ctypes.data, config_order, out.struct(), n_threads or threads())
    if rc != abi.OK:
        raise RuntimeError(f"oracle status {rc}")
    return out
