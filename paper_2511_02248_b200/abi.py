"""ctypes mirror of include/opscale_b200.h (structs and constants).

Kept byte-for-byte in step with the header; tests/test_abi.py checks the
struct sizes against the ones the compiled library reports.
"""

import ctypes as C

ABI_VERSION = 1
MAX_OPS = 32
MAX_EDGES = 256
MAX_P = 8
MAX_DEVICES = 1024
PRED_FIELDS = 7

OK, ERR_ARG, ERR_CUDA, ERR_SPACE, ERR_NODEVICE = 0, 1, 2, 3, 4

W_NO_STABLE_BOUNDS = 0x1
W_NO_STABLE_PARAMS = 0x2
W_NO_STABLE_MODEL = 0x4
W_ZERO_DIVISION = 0x8
W_UNSTABLE_ROUNDING = 0x10
W_FLEET_EXHAUSTED = 0x20
W_INFEASIBLE_PLACEMENT = 0x40
W_IDLE = 0x80
W_NO_STABLE_INIT = 0x100
W_TRACE_TRUNCATED = 0x200
W_ORDER_SENSITIVE = 0x400  # opt-in brute-force certificate: decision may depend on the leaf-sum order
W_INIT_OP_SHIFT = 16     # 1 + dag.node_ids position of the op init_configs names
W_BOUNDS_OP_SHIFT = 22   # 1 + lex rank of the op without a finite menu entry
W_OP_FIELD = 0x3F

ACT_UPSCALE, ACT_DOWNSCALE, ACT_HEADROOM, ACT_PRUNE, ACT_RESEED = 1, 2, 3, 4, 5
ACTION_NAMES = {1: "upscale", 2: "downscale", 3: "headroom", 4: "prune", 5: "reseed_uniform"}

MODE_ORACLE = 0
MODE_MODEL = 1
MODE_OPERATOR = 2
PLAN_CERTIFY = 0x100       # OR'ed into the host-buffer mode: run the order certificate (brute force)
CERTIFY_BAND_ULPS = 64.0

KEY_INFEASIBLE = 0x7FFFFFFFFFFFFFFF
KEY_LEX_BITS = 40

_D = C.c_double
_I = C.c_int32
_U = C.c_uint32


class OpscDag(C.Structure):
    _fields_ = [
        ("n_ops", _I), ("n_edges", _I),
        ("topo", _I * MAX_OPS), ("node_order", _I * MAX_OPS),
        ("layer_count", _I * MAX_OPS), ("pred_mask", _U * MAX_OPS),
        ("sink_mask", _U), ("has_phase", _U * 2),
        ("c0", (_D * MAX_OPS) * 2), ("c1", (_D * MAX_OPS) * 2), ("c2", (_D * MAX_OPS) * 2),
        ("eta", _D * MAX_OPS), ("weight_mem", _D * MAX_OPS), ("m0", _D * MAX_OPS),
        ("m1", _D * MAX_OPS), ("s0", _D * MAX_OPS), ("s1", _D * MAX_OPS),
        ("out_ptr", _I * (MAX_OPS + 1)),
        ("out_v0", _D * MAX_EDGES), ("out_v1", _D * MAX_EDGES),
        ("link_bw", _D),
    ]


class OpscGrid(C.Structure):
    _fields_ = [
        ("r_max", _I), ("n_p", _I * MAX_OPS), ("p_vals", (_I * MAX_P) * MAX_OPS),
        ("b_max", _I * MAX_OPS), ("menu_off", _I * (MAX_OPS + 1)),
        ("r_cap", _I), ("params_n_p", _I * MAX_OPS),
        ("params_p_vals", (_I * MAX_P) * MAX_OPS), ("params_b_max", _I * MAX_OPS),
    ]


class OpscModelSpec(C.Structure):
    _fields_ = [("p_base", _I * MAX_OPS), ("b_cap", _I), ("r_cap", _I)]


class OpscGreedySpec(C.Structure):
    _fields_ = [("n_p", _I * MAX_OPS), ("p_vals", (_I * MAX_P) * MAX_OPS),
                ("b_max", _I * MAX_OPS), ("r_cap", _I), ("max_iterations", _I),
                ("prune_excess_replicas", _I), ("model", OpscModelSpec)]


class OpscTraceEntry(C.Structure):
    _fields_ = [("latency", _D), ("objective", _I), ("to_r", C.c_int16), ("to_b", C.c_int16),
                ("to_p", C.c_int16), ("op", C.c_int8), ("action", C.c_uint8),
                ("reserved", C.c_int32)]


class OpscPlaceSpec(C.Structure):
    _fields_ = [("n_devices", _I), ("uniform_cap", _I), ("alpha", _D), ("beta", _D),
                ("mem_cap", C.c_void_p)]


class OpscWindows(C.Structure):
    _fields_ = [("n", _I), ("qps", C.c_void_p), ("seq_len", C.c_void_p),
                ("phase", C.c_void_p), ("slo", C.c_void_p), ("eps", C.c_void_p)]


class OpscDecisions(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "key", "cfg", "feasible", "status", "latency", "objective", "path",
        "pred", "stable", "energy", "memory", "devices")] + [
        ("trace_cap", _I), ("trace_len", C.c_void_p), ("trace", C.c_void_p)]


class OpscTraceRecords(C.Structure):
    _fields_ = [("n", C.c_int64), ("arrival", C.c_void_p), ("input_len", C.c_void_p),
                ("output_len", C.c_void_p)]


class OpscPlaceShared(C.Structure):
    _fields_ = [("n_devices", _I), ("mem_cap", C.c_void_p), ("compute_cap", C.c_void_p),
                ("slo", _D), ("slack_weight_mem", _D), ("slack_weight_compute", _D),
                ("max_sm_load", _D), ("theta", _D), ("exponent", _D), ("alpha", _D), ("beta", _D),
                ("flags", _I)]


MAX_PEERS = 8
IPC_HANDLE_BYTES = 64

PLACE_DEFAULT_STREAM = 0x1
PLACE_WINDOW_SLO = 0x2


class OpscPlacement(C.Structure):
    _fields_ = [("cap_assign", _I), ("cap_dev", _I)] + [(name, C.c_void_p) for name in (
        "n_assign", "devices_used", "feasible", "status", "latency", "energy", "memory",
        "a_op", "a_replica", "a_device", "a_share", "a_latency", "d_mem", "d_sm", "d_energy")]
