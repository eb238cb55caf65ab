"""Golden vectors for reference-valid inputs outside the main sets: slo = +inf
(AutoscaleParams only requires slo > 0, autoscaler.py:113-116), menus past
the GPU's shared-memory tile, and per-operator dict b_max / parallelism
(autoscaler.py:106-107, 120-131; bounds inheriting them). Runs the reference planners
from /root/reference in this container and writes edges_{oracle,model,greedy}.json
in the same record format as make_golden.py.

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONHASHSEED=0 \
        python tests/golden/make_golden_edges.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as M  # noqa: E402

INF = float("inf")


def oracle_cases():
    cases = []
    for qps in (8.0, 30.0, 60.0):
        cases.append(dict(name=f"edge/slo_inf/cfg1/q{qps:g}", scenario="cfg1",
                          point=dict(qps=qps, seq_len=4096, phase="prefill"), params=dict(slo=INF),
                          bounds=dict(r_max=3, b_max=2, parallelism=[1, 2])))
    cases.append(dict(name="edge/slo_inf/cfg1/decode", scenario="cfg1",
                      point=dict(qps=60.0, seq_len=2048, phase="decode"), params=dict(slo=INF),
                      bounds=dict(r_max=2, b_max=3, parallelism=[1, 2])))
    # menus too large for the shared-memory tile (the flat compose kernel):
    # one operator with a 65536-entry menu, two operators with 8192 x 16
    one = {"nodes": [{"id": "solo", "kind": "linear", "layer_count": 32, "profile_ref": "mlp"}],
           "edges": []}
    c7, p7 = M.S.SCENARIOS["cfg1"]
    cases.append(dict(name="edge/large_menu/single_op_65536", dag=one, profiles=p7,
                      point=dict(qps=300.0, seq_len=2048, phase="prefill"), params=dict(slo=0.05),
                      bounds=dict(r_max=512, b_max=32, parallelism=[1, 2, 4, 8])))
    two = {"nodes": [{"id": "b2", "kind": "linear", "layer_count": 32, "profile_ref": "mlp"},
                     {"id": "a1", "kind": "attention", "layer_count": 32, "profile_ref": "attn"}],
           "edges": [{"src": "b2", "dst": "a1", "volume_ref": "mlp"}]}
    cases.append(dict(name="edge/large_menu/two_op", dag=two, profiles=p7,
                      point=dict(qps=120.0, seq_len=2048, phase="prefill"), params=dict(slo=0.3),
                      bounds=dict(r_max=256, b_max=16, parallelism=[1, 2])))
    cases.append(dict(name="edge/slo_inf/nostable_bounds", scenario="cfg1",
                      point=dict(qps=40.0, seq_len=4096, phase="prefill"), params=dict(slo=INF),
                      bounds=dict(r_max=1, b_max=1, parallelism=[1])))
    return cases + dict_cases(True)


# per-operator b_max / parallelism (AutoscaleParams accepts dicts,
# autoscaler.py:106-107, 120-131; brute-force bounds inherit them when None)
OPS7 = ["embed", "norm", "qkv", "attn", "mlp", "act"]
DICT_PARAMS = [
    dict(slo=0.5, b_max={"embed": 4, "norm": 2, "qkv": 3, "attn": 1, "mlp": 2, "act": 5},
         parallelism={"embed": (1,), "norm": (1, 2), "qkv": (2, 1), "attn": (1, 2, 4), "mlp": (4, 2), "act": (1,)}),
    dict(slo=0.2, epsilon=0.02, b_max={"embed": 8, "norm": 8, "qkv": 16, "attn": 4, "mlp": 32, "act": 8},
         parallelism={"embed": (1, 2), "norm": (1,), "qkv": (1, 2, 4, 8), "attn": (2, 4), "mlp": (1, 8), "act": (1, 2)}),
]


# brute force enumerates literally on the CPU oracle: keep the inherited grid small
DICT_PARAMS_BF = [
    DICT_PARAMS[0],
    dict(slo=0.2, epsilon=0.02, b_max={"embed": 2, "norm": 1, "qkv": 3, "attn": 2, "mlp": 2, "act": 1},
         parallelism={"embed": (1, 2), "norm": (1,), "qkv": (1, 2, 4), "attn": (2, 4), "mlp": (1, 8), "act": (1, 2)}),
]


def dict_cases(with_bounds):
    out = []
    for i, kw in enumerate(DICT_PARAMS_BF if with_bounds else DICT_PARAMS):
        for q in (20.0, 90.0):
            c = dict(name=f"edge/dict_params/{i}/q{q:g}", scenario="cfg1",
                     point=dict(qps=q, seq_len=1024, phase="prefill"), params=dict(kw))
            if with_bounds:
                c["bounds"] = dict(r_max=3, b_max=None, parallelism=None)
            out.append(c)
    return out


def model_cases():
    return [dict(name=f"edge/slo_inf/{cfg}/{ph}", scenario=cfg,
                 point=dict(qps=q, seq_len=2048, phase=ph), params=dict(slo=INF))
            for cfg, q in (("cfg1", 30.0), ("cfg2", 12.0)) for ph in ("prefill", "decode")] + dict_cases(False)


def greedy_cases():
    # large batch bounds: init_configs over B in several 64-wide chunks, and
    # move sets (B x distinct P) past one 512-move chunk
    big = [dict(name=f"edge/greedy_big_b/{b}/{ph}", scenario="cfg1",
                point=dict(qps=q, seq_len=1024, phase=ph), params=dict(slo=slo, b_max=b, epsilon=slo * 0.05))
           for b, ph, q, slo in ((100, "prefill", 120.0, 0.3), (200, "decode", 3000.0, 0.05),
                                 (160, "prefill", 400.0, 0.2))]
    return [dict(name=f"edge/slo_inf/{cfg}/{ph}", scenario=cfg,
                 point=dict(qps=q, seq_len=2048, phase=ph), params=dict(slo=INF))
            for cfg, q in (("cfg1", 30.0), ("cfg2", 12.0)) for ph in ("prefill", "decode")] + dict_cases(False) + big


def case_inputs(c):
    """make_golden.case_inputs plus per-op dicts and None bounds fields."""
    if "scenario" in c:
        dag_spec, prof = M.S.SCENARIOS[c["scenario"]]
    else:
        dag_spec, prof = c["dag"], c["profiles"]
    pt = M.ref.WorkloadPoint(c["point"]["qps"], c["point"]["seq_len"], c["point"]["phase"])
    kw = dict(c["params"])
    if "parallelism" in kw:
        par = kw["parallelism"]
        kw["parallelism"] = {k: tuple(v) for k, v in par.items()} if isinstance(par, dict) else tuple(par)
    params = M.ref.AutoscaleParams(**kw)
    bounds = None
    if "bounds" in c:
        b = dict(c["bounds"])
        if b.get("parallelism") is not None:
            b["parallelism"] = tuple(b["parallelism"])
        bounds = M.ref.BruteForceBounds(**b)
    return dag_spec, prof, pt, params, bounds


def serialise_case(c, pt, params, bounds):
    out = {"name": c["name"]}
    if "scenario" in c:
        out["scenario"] = c["scenario"]
    else:
        out["dag"], out["profiles"] = c["dag"], c["profiles"]
    out["point"] = M.point_json(pt)
    par = params.parallelism
    out["params"] = {"slo": M.H(params.slo), "epsilon": M.H(params.epsilon), "b_max": params.b_max,
                     "parallelism": {k: list(v) for k, v in par.items()} if isinstance(par, dict) else list(par),
                     "r_cap": params.r_cap, "max_iterations": params.max_iterations,
                     "prune_excess_replicas": params.prune_excess_replicas}
    if bounds is not None:
        out["bounds"] = {"r_max": bounds.r_max, "b_max": bounds.b_max,
                         "parallelism": None if bounds.parallelism is None else list(bounds.parallelism)}
    return out


def main():
    out = []
    for c in oracle_cases():
        dag_spec, prof, pt, params, bounds = case_inputs(c)
        j, plan, dag, profiles = M.run_oracle(dag_spec, prof, pt, params, bounds)
        rec = serialise_case(c, pt, params, bounds)
        rec["expected"] = j
        if plan is not None:
            rec["metrics"] = M.metrics_json(plan, dag, profiles, pt, 256, 180e9)
            rec["metrics_small_fleet"] = M.metrics_json(plan, dag, profiles, pt, 4, 40e9)
            rec["metrics_tiny_cap"] = M.metrics_json(plan, dag, profiles, pt, 64, 2.0e8)
        rec["hash_sensitive"] = False
        out.append(rec)
    json.dump(out, open(os.path.join(HERE, "edges_oracle.json"), "w"), separators=(",", ":"))
    model = []
    for c in model_cases():
        dag_spec, prof, pt, params, _ = case_inputs(c)
        j, plan, dag, profiles = M.run_model(dag_spec, prof, pt, params)
        rec = serialise_case(c, pt, params, None)
        rec["expected"] = j
        if plan is not None:
            rec["metrics"] = M.metrics_json(plan, dag, profiles, pt, 4096, 180e9)
        model.append(rec)
    json.dump(model, open(os.path.join(HERE, "edges_model.json"), "w"), separators=(",", ":"))
    greedy = []
    for c in greedy_cases():
        dag_spec, prof, pt, params, _ = case_inputs(c)
        j, plan, dag, profiles = M.run_greedy(dag_spec, prof, pt, params)
        rec = serialise_case(c, pt, params, None)
        rec["expected"] = j
        if plan is not None:
            rec["metrics"] = M.metrics_json(plan, dag, profiles, pt, 4096, 180e9)
        greedy.append(rec)
    json.dump(greedy, open(os.path.join(HERE, "edges_greedy.json"), "w"), separators=(",", ":"))
    for name, recs in (("oracle", out), ("model", model), ("greedy", greedy)):
        print(name, [(r["name"], r["expected"].get("error") or (r["expected"]["objective"],
                                                                 r["expected"]["feasible"])) for r in recs])


if __name__ == "__main__":
    main()
