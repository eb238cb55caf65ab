"""Synthetic planning scenarios for the BASELINE.json configs.

The reference's bundled DAG/profile packs are absent,
so the scenarios are defined here as plain JSON-style dicts in the
reference's own schemas (DAG: opgraph.py:151-171; profiles:
perfmodel.py:300-324). Both the reference and this package build their
objects from the same dicts, which is what lets the golden fixtures of
tests/golden/ pin decisions on identical inputs.

  cfg1  Llama-2-7B 6-op chain, one bursty 60 s window, small exhaustive grid
  cfg2  Llama-2-70B 10-op chain, 1 h bursty trace, 60 s windows
  cfg3  multimodal DAG (vision branch + text embed merging into the LLM),
        heavy-tailed lengths; `multimodal_small` is a <=6-op variant the
        reference brute force accepts
  cfg5  the cfg1 DAG over a 24 h trace (1440 prefill windows) with a ~1e8
        candidate grid per window

Window statistics of every trace (qps, seq_len per window and phase) were
produced by the reference's synth_workload + windowize and are stored in
workloads/traces.npz by tests/golden/make_traces.py; the package's
`workload.py` regenerates them bit-identically.

Bench and test data only: nothing in the product package
(paper_2511_02248_b200/) imports this module.
"""

from __future__ import annotations

import os

import numpy as np

from paper_2511_02248_b200.model import build_dag, profiles_from_dict

_DATA = os.path.dirname(os.path.abspath(__file__))


def _chain(spec):
    nodes = [{"id": i, "kind": k, "layer_count": n, "profile_ref": i} for i, k, n in spec]
    edges = [{"src": a[0], "dst": b[0], "volume_ref": a[0]} for a, b in zip(spec, spec[1:])]
    return {"nodes": nodes, "edges": edges}


# ---------------------------------------------------------------- Llama-2-7B

DAG_7B = _chain([
    ("embed", "embedding", 1), ("norm", "norm", 64), ("qkv", "linear", 32),
    ("attn", "attention", 32), ("mlp", "linear", 32), ("act", "activation", 32),
])


def _op(pre, dec, w=0.0, m1=0.0, v1=0.0, s=(0.0, 0.0), kind="other", m0=0.0, v0=0.0):
    c = lambda t: {"c0": t[0], "c1": t[1], "c2": t[2] if len(t) > 2 else 0.0}
    return {"prefill": c(pre), "decode": c(dec), "weight_mem": w, "m0": m0, "m1": m1,
            "v0": v0, "v1": v1, "s0": s[0], "s1": s[1], "eta": 0.9, "kind": kind}


# SURVEY.md Appendix C table, with the B200 NVLink 5 per-direction bandwidth.
PROFILES_7B = {
    "_link_bandwidth": 900e9,
    "_interference": {"theta": 0.5, "exponent": 1.0},
    "embed": _op((1e-5, 2e-9), (1e-5, 2e-9), 2.6e8, 8192, 8192, (.05, 1e-5), "embedding"),
    "norm": _op((5e-6, 4e-9), (5e-6, 4e-9), 8e3, 8192, 8192, (.05, 2e-5), "norm"),
    "qkv": _op((1e-5, 1.2e-7), (2e-5, 1.5e-7), 1.0e8, 24576, 24576, (.2, 4e-4), "linear"),
    "attn": _op((1e-5, 2e-8, 1.5e-10), (2e-5, 1e-7), 0.0, 16384, 8192, (.3, 5e-4), "attention"),
    "mlp": _op((1e-5, 3.5e-7), (3e-5, 4e-7), 2.7e8, 44000, 8192, (.3, 6e-4), "linear"),
    "act": _op((4e-6, 3e-9), (4e-6, 3e-9), 0.0, 22000, 22000, (.05, 2e-5), "activation"),
}

# ---------------------------------------------------------------- Llama-2-70B

DAG_70B = _chain([
    ("embed", "embedding", 1), ("norm_attn", "norm", 80), ("qkv", "linear", 80),
    ("attn", "attention", 80), ("o_proj", "linear", 80), ("norm_mlp", "norm", 80),
    ("gate_up", "linear", 80), ("act", "activation", 80), ("down", "linear", 80),
    ("lm_head", "linear", 1),
])


def _lin(c1p, c1d, w):
    return _op((1e-5, c1p), (2e-5, c1d), w, 65536, 16384, (.3, 6e-4), "linear")


PROFILES_70B = {
    "_link_bandwidth": 900e9,
    "_interference": {"theta": 0.5, "exponent": 1.0},
    "embed": _op((1e-5, 2e-9), (1e-5, 2e-9), 5.2e8, 16384, 16384, (.05, 1e-5), "embedding"),
    "norm_attn": _op((5e-6, 6e-9), (5e-6, 6e-9), 1.6e4, 16384, 16384, (.05, 2e-5), "norm"),
    "norm_mlp": _op((5e-6, 6e-9), (5e-6, 6e-9), 1.6e4, 16384, 16384, (.05, 2e-5), "norm"),
    "qkv": _lin(2.0e-7, 2.5e-7, 2.0e8),
    "attn": _op((1e-5, 3e-8, 2.5e-10), (2e-5, 1.5e-7), 0.0, 32768, 16384, (.3, 5e-4), "attention"),
    "o_proj": _lin(1.6e-7, 2.0e-7, 1.3e8),
    "gate_up": _lin(1.1e-6, 1.3e-6, 1.2e9),
    "act": _op((4e-6, 5e-9), (4e-6, 5e-9), 0.0, 57344, 57344, (.05, 2e-5), "activation"),
    "down": _lin(5.5e-7, 6.5e-7, 5.9e8),
    "lm_head": _lin(8e-7, 9e-7, 1.0e9),
}

# ---------------------------------------------------------------- multimodal


def _dag(nodes, edges):
    return {
        "nodes": [{"id": i, "kind": k, "layer_count": n, "profile_ref": i} for i, k, n in nodes],
        "edges": [{"src": a, "dst": b, "volume_ref": a} for a, b in edges],
    }


DAG_MM = _dag(
    [("patch_embed", "embedding", 1), ("vit_attn", "attention", 32), ("vit_mlp", "linear", 32),
     ("projector", "linear", 1), ("embed", "embedding", 1), ("norm", "norm", 64),
     ("qkv", "linear", 32), ("attn", "attention", 32), ("o_proj", "linear", 32),
     ("mlp", "linear", 32), ("act", "activation", 32), ("lm_head", "linear", 1)],
    [("patch_embed", "vit_attn"), ("vit_attn", "vit_mlp"), ("vit_mlp", "projector"),
     ("projector", "norm"), ("embed", "norm"), ("norm", "qkv"), ("qkv", "attn"),
     ("attn", "o_proj"), ("o_proj", "mlp"), ("mlp", "act"), ("act", "lm_head")],
)

PROFILES_MM = {
    "_link_bandwidth": 900e9,
    "_interference": {"theta": 0.5, "exponent": 1.0},
    "patch_embed": _op((8e-6, 3e-9), (8e-6, 3e-9), 1.2e7, 6144, 6144, (.1, 2e-5), "embedding"),
    "vit_attn": _op((1e-5, 1.5e-8, 1.2e-10), (1.5e-5, 6e-8), 0.0, 12288, 6144, (.25, 4e-4), "attention"),
    "vit_mlp": _op((1e-5, 1.8e-7), (2e-5, 2.2e-7), 1.1e8, 24576, 6144, (.25, 5e-4), "linear"),
    "projector": _op((6e-6, 4e-8), (8e-6, 5e-8), 2.0e7, 8192, 8192, (.1, 1e-4), "linear"),
    "embed": PROFILES_7B["embed"],
    "norm": PROFILES_7B["norm"],
    "qkv": PROFILES_7B["qkv"],
    "attn": PROFILES_7B["attn"],
    "o_proj": _op((1e-5, 9e-8), (2e-5, 1.1e-7), 6.7e7, 16384, 8192, (.2, 4e-4), "linear"),
    "mlp": PROFILES_7B["mlp"],
    "act": PROFILES_7B["act"],
    "lm_head": _op((1e-5, 5e-7), (2e-5, 6e-7), 2.6e8, 65536, 8192, (.3, 6e-4), "linear"),
}

DAG_MM_SMALL = _dag(
    [("patch_embed", "embedding", 1), ("vit", "attention", 32), ("projector", "linear", 1),
     ("embed", "embedding", 1), ("llm_attn", "attention", 32), ("llm_mlp", "linear", 32)],
    [("patch_embed", "vit"), ("vit", "projector"), ("projector", "llm_attn"),
     ("embed", "llm_attn"), ("llm_attn", "llm_mlp")],
)

PROFILES_MM_SMALL = {
    "_link_bandwidth": 900e9,
    "_interference": {"theta": 0.5, "exponent": 1.0},
    "patch_embed": PROFILES_MM["patch_embed"],
    "vit": PROFILES_MM["vit_attn"],
    "projector": PROFILES_MM["projector"],
    "embed": PROFILES_7B["embed"],
    "llm_attn": PROFILES_7B["attn"],
    "llm_mlp": PROFILES_7B["mlp"],
}

# ---------------------------------------------------------------- traces

# SynthSpec keyword sets (workload.py:161-192) and windowing per config.
TRACES = {
    "cfg1": dict(spec=dict(kind="burst", rate=8.0, duration=60.0, burst_factor=4.0,
                           burst_duty=0.2, input_len_median=1024.0, input_len_sigma=0.8),
                 seed=0, window_len=60.0, quantile=0.95),
    "cfg2": dict(spec=dict(kind="burst", rate=8.0, duration=3600.0, period=600.0,
                           burst_factor=4.0, burst_duty=0.2, input_len_median=1024.0,
                           input_len_sigma=0.8, output_len_median=256.0,
                           output_len_sigma=0.6),
                 seed=0, window_len=60.0, quantile=0.95),
    "cfg3": dict(spec=dict(kind="diurnal", rate=6.0, duration=3600.0, period=3600.0,
                           amplitude=0.5, input_len_median=768.0, input_len_sigma=1.5,
                           output_len_median=192.0, output_len_sigma=1.2),
                 seed=1, window_len=60.0, quantile=0.95),
    "cfg5": dict(spec=dict(kind="diurnal", rate=8.0, duration=86400.0, period=86400.0,
                           amplitude=0.6, input_len_median=1024.0, input_len_sigma=0.8,
                           output_len_median=256.0, output_len_sigma=0.6),
                 seed=5, window_len=60.0, quantile=0.95),
}

# SLOs (TTFT for prefill, TBT for decode) and candidate grids per config.
SLO = {
    "cfg1": {"prefill": 0.5, "decode": 0.05},
    "cfg2": {"prefill": 2.0, "decode": 0.15},
    "cfg3": {"prefill": 1.0, "decode": 0.08},
    "cfg3s": {"prefill": 1.0, "decode": 0.08},
    "cfg5": {"prefill": 0.5, "decode": 0.05},
}
GRIDS = {
    "cfg1": dict(r_max=3, b_max=2, parallelism=(1, 2)),     # 12^6  ~ 3.0e6
    "cfg2": dict(r_max=3, b_max=1, parallelism=(2, 4)),     # 6^10  ~ 6.0e7 (96/120 windows feasible)
    "cfg3": dict(r_max=3, b_max=1, parallelism=(1, 2)),     # 6^12  ~ 2.2e9 (sharded / sampled)
    "cfg3s": dict(r_max=3, b_max=2, parallelism=(1, 2)),    # 12^6 on the 6-op variant
    "cfg5": dict(r_max=4, b_max=3, parallelism=(1, 2)),     # 24^6  ~ 1.9e8
}

SCENARIOS = {
    "cfg1": (DAG_7B, PROFILES_7B),
    "cfg2": (DAG_70B, PROFILES_70B),
    "cfg3": (DAG_MM, PROFILES_MM),
    "cfg3s": (DAG_MM_SMALL, PROFILES_MM_SMALL),
    "cfg5": (DAG_7B, PROFILES_7B),
}


def scenario(name):
    """(OperatorDag, ProfileSet) built with this package's mirror types."""
    dag_spec, prof = SCENARIOS[name]
    return build_dag(dag_spec), profiles_from_dict(prof)


def trace_windows(name):
    """Per-window stats of a config's trace as arrays:
    dict(prefill_qps, prefill_len, decode_qps, decode_len, t0, t1)."""
    key = "cfg3" if name == "cfg3s" else name
    with np.load(os.path.join(_DATA, "traces.npz")) as z:
        return {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(key + "/")}
