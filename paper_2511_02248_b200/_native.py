"""ctypes binding of libopscale_b200.so (the C ABI in include/opscale_b200.h).

The planner search has no CPU implementation in this package: if the
library is missing or no CUDA device is visible, every entry point raises
DeviceUnavailable.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import abi, tables
from .errors import DeviceUnavailable, SearchSpaceTooLarge

HERE = os.path.dirname(os.path.abspath(__file__))
# OPSC_LIB_PATH: dev-only override for same-box A/B timing of two builds
LIB_PATH = os.environ.get("OPSC_LIB_PATH") or os.path.join(HERE, "_lib", "libopscale_b200.so")

# every symbol include/opscale_b200.h declares
EXPORTS = (
    "opsc_abi_version", "opsc_status_string", "opsc_device_count", "opsc_menu_build",
    "opsc_stability_check", "opsc_compose_argmin", "opsc_fill_keys", "opsc_init_windows",
    "opsc_menu_fallback",
    "opsc_decode_decisions", "opsc_model_grid", "opsc_materialize", "opsc_ctx_create",
    "opsc_ctx_destroy", "opsc_plan_windows_host", "opsc_ctx_last_launches", "opsc_ctx_last_ms", "opsc_fp64_peak",
    "opsc_compose_boundary",
    "opsc_candidate_probe", "opsc_greedy", "opsc_windowize", "opsc_windowize_workspace",
    "opsc_greedy_state_bytes", "opsc_greedy_phase", "opsc_model_table_bytes",
    "opsc_model_grid_table", "opsc_place_shared_workspace", "opsc_place_shared",
    "opsc_ipc_alloc", "opsc_ipc_open", "opsc_ipc_close", "opsc_ipc_free",
    "opsc_compose_argmin_peers", "opsc_peer_barrier", "opsc_copy_keys",
    "opsc_certify_workspace", "opsc_certify_order", "opsc_menu_stability", "opsc_decode_materialize",
    "opsc_interference_pow",
)

_lib = None
_lock = threading.Lock()
_tls = threading.local()


def load():
    """Load the library and declare signatures (no CUDA call is made)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(
                f"{LIB_PATH} is not built; run `python -m paper_2511_02248_b200.build`")
        L = C.CDLL(LIB_PATH)
        P, I = C.c_void_p, C.c_int32
        W, D = abi.OpscWindows, abi.OpscDecisions
        sig = {
            "opsc_abi_version": ([], C.c_int),
            "opsc_status_string": ([C.c_int], C.c_char_p),
            "opsc_device_count": ([P], C.c_int),
            "opsc_menu_build": ([P, P, W, P, P, P], C.c_int),
            "opsc_stability_check": ([P, P, W, P, P], C.c_int),
            "opsc_compose_argmin": ([P, P, W, P, I, I, P, P], C.c_int),
            "opsc_fill_keys": ([P, I, P], C.c_int),
            "opsc_init_windows": ([W, P, P, P, P], C.c_int),
            "opsc_menu_fallback": ([P, P, I, P, P, P], C.c_int),
            "opsc_decode_decisions": ([P, P, I, P, P, P, P, P, P], C.c_int),
            "opsc_model_grid": ([P, P, W, P, P, P, P], C.c_int),
            "opsc_materialize": ([P, W, I, P, D, P], C.c_int),
            "opsc_ctx_create": ([I, I, P], C.c_int),
            "opsc_ctx_destroy": ([P], C.c_int),
            "opsc_plan_windows_host": ([P, I, P, P, P, P, P, W, D], C.c_int),
            "opsc_greedy": ([P, P, W, P, P, P, D, P], C.c_int),
            "opsc_windowize_workspace": ([C.c_int64, I], C.c_size_t),
            "opsc_greedy_state_bytes": ([I], C.c_size_t),
            "opsc_model_table_bytes": ([P, I, I], C.c_size_t),
            "opsc_place_shared_workspace": ([I, I, I, I], C.c_size_t),
            "opsc_place_shared": ([P, P, W, P, P, I, abi.OpscPlacement, P, C.c_size_t, P], C.c_int),
            "opsc_model_grid_table": ([P, P, W, P, P, P, P, C.c_size_t, P], C.c_int),
            "opsc_greedy_phase": ([P, P, W, I, P, P, P, P, D, P], C.c_int),
            "opsc_windowize": ([abi.OpscTraceRecords, C.c_double, C.c_double, I, P, P, P, P, P,
                                C.c_size_t, P], C.c_int),
            "opsc_ctx_last_launches": ([P, P], C.c_int),
            "opsc_ctx_last_ms": ([P, P], C.c_int),
            "opsc_compose_boundary": ([P, P, abi.OpscWindows, P, C.c_double, P, P], C.c_int),
            "opsc_fp64_peak": ([I, P, P, P], C.c_int),
            "opsc_candidate_probe": ([I, I, P, P, P], C.c_int),
            "opsc_ipc_alloc": ([C.c_size_t, P, P], C.c_int),
            "opsc_ipc_open": ([P, P], C.c_int),
            "opsc_ipc_close": ([P], C.c_int),
            "opsc_ipc_free": ([P], C.c_int),
            "opsc_compose_argmin_peers": ([P, P, W, P, I, I, P, I, P], C.c_int),
            "opsc_peer_barrier": ([P, I, I, C.c_uint32, I, P, P], C.c_int),
            "opsc_copy_keys": ([P, P, I, P], C.c_int),
            "opsc_certify_workspace": ([I], C.c_size_t),
            "opsc_certify_order": ([P, P, W, P, C.c_double, P, C.c_size_t, P, P], C.c_int),
            "opsc_menu_stability": ([P, P, W, P, P, P], C.c_int),
            "opsc_decode_materialize": ([P, P, W, P, P, P, D, P], C.c_int),
            "opsc_interference_pow": ([P, P, P, C.c_int64, P], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        if L.opsc_abi_version() != abi.ABI_VERSION:
            raise DeviceUnavailable("libopscale_b200.so ABI version mismatch; rebuild it")
        _lib = L
        return L


def ref(x):
    return C.cast(C.byref(x), C.c_void_p)


def check(rc, what):
    if rc == abi.OK:
        return
    msg = load().opsc_status_string(rc).decode()
    if rc == abi.ERR_SPACE:
        raise SearchSpaceTooLarge(f"{what}: {msg}")
    if rc == abi.ERR_NODEVICE:
        raise DeviceUnavailable(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def device_count():
    n = C.c_int(0)
    load().opsc_device_count(C.cast(C.byref(n), C.c_void_p))
    return n.value


class Context:
    """Owns an OpscContext (stream + device workspace) for host-buffer calls."""

    def __init__(self, device=0, max_windows=0):
        L = load()
        if device_count() <= device:
            raise DeviceUnavailable("no CUDA device visible: the planner search runs only on the GPU")
        self._p = C.c_void_p()
        check(L.opsc_ctx_create(device, max_windows, C.cast(C.byref(self._p), C.c_void_p)),
              "opsc_ctx_create")

    def close(self):
        if self._p:
            load().opsc_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._p

    def last_launches(self):
        n = C.c_int32(0)
        check(load().opsc_ctx_last_launches(self._p, C.cast(C.byref(n), C.c_void_p)), "launches")
        return n.value

    def last_ms(self):
        """Device time of the last plan_windows call (first H2D .. last D2H)."""
        ms = C.c_float(0.0)
        check(load().opsc_ctx_last_ms(self._p, C.cast(C.byref(ms), C.c_void_p)), "last_ms")
        return ms.value

    def plan_windows(self, mode, problem, windows, grid=None, model=None, place=None, out=None,
                     greedy=None, trace_cap=4096, certify=False):
        place = place or tables.pack_place()
        if out is None:
            out = tables.DecisionArrays(windows.n, problem.n_ops,
                                        trace_cap if mode == abi.MODE_OPERATOR else 0)
        g = grid if grid is not None else _EMPTY[0]
        m = model if model is not None else _EMPTY[1]
        gs = greedy if greedy is not None else _EMPTY[2]
        A = C.addressof
        flags = abi.PLAN_CERTIFY if certify and mode == abi.MODE_ORACLE else 0
        rc = load().opsc_plan_windows_host(self._p, mode | flags, A(problem.table), A(g), A(m), A(gs),
                                           A(place.spec), windows.struct(), out.struct())
        check(rc, "opsc_plan_windows_host")
        return out


_EMPTY = (abi.OpscGrid(), abi.OpscModelSpec(), abi.OpscGreedySpec())  # read-only placeholders


def context():
    """Per-thread context: concurrent planner calls never share a stream."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context()
        _tls.ctx = ctx
    return ctx


def plan_windows_host(mode, problem, windows, grid=None, model=None, place=None, greedy=None,
                      trace_cap=4096, out=None, certify=False):
    """One host-buffer planning call on this thread's context. Greedy move
    traces have no length limit in the reference (max_iterations per loop plus
    headroom / prune entries, autoscaler.py:391, 446-587): windows whose
    trace outgrew `trace_cap` (the kernel keeps counting past the cap) are
    re-planned with room for their whole trace -- the planner is
    deterministic, so only the trace rows change."""
    ctx = context()
    out = ctx.plan_windows(mode, problem, windows, grid=grid, model=model, place=place,
                           greedy=greedy, trace_cap=trace_cap, out=out, certify=certify)
    if mode == abi.MODE_OPERATOR and out.trace_cap:
        import numpy as np
        cut = np.nonzero(out.status & abi.W_TRACE_TRUNCATED)[0]
        if len(cut):
            cap = int(out.trace_len[cut].max())
            again = ctx.plan_windows(mode, problem, windows.take(cut), grid=grid, model=model,
                                     place=place, greedy=greedy, trace_cap=cap)
            out = out.with_trace_cap(cap)
            out.splice(cut, again)
    return out
