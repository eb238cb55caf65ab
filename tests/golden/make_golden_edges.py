"""Golden vectors for slo = +inf (the reference accepts it: AutoscaleParams
only requires slo > 0, autoscaler.py:113-116). Runs the reference planners
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
    return cases


def model_cases():
    return [dict(name=f"edge/slo_inf/{cfg}/{ph}", scenario=cfg,
                 point=dict(qps=q, seq_len=2048, phase=ph), params=dict(slo=INF))
            for cfg, q in (("cfg1", 30.0), ("cfg2", 12.0)) for ph in ("prefill", "decode")]


def greedy_cases():
    return [dict(name=f"edge/slo_inf/{cfg}/{ph}", scenario=cfg,
                 point=dict(qps=q, seq_len=2048, phase=ph), params=dict(slo=INF))
            for cfg, q in (("cfg1", 30.0), ("cfg2", 12.0)) for ph in ("prefill", "decode")]


def main():
    out = []
    for c in oracle_cases():
        dag_spec, prof, pt, params, bounds = M.case_inputs(c)
        j, plan, dag, profiles = M.run_oracle(dag_spec, prof, pt, params, bounds)
        rec = M.serialise_case(c, pt, params, bounds)
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
        dag_spec, prof, pt, params, _ = M.case_inputs(c)
        j, plan, dag, profiles = M.run_model(dag_spec, prof, pt, params)
        rec = M.serialise_case(c, pt, params, None)
        rec["expected"] = j
        if plan is not None:
            rec["metrics"] = M.metrics_json(plan, dag, profiles, pt, 4096, 180e9)
        model.append(rec)
    json.dump(model, open(os.path.join(HERE, "edges_model.json"), "w"), separators=(",", ":"))
    greedy = []
    for c in greedy_cases():
        dag_spec, prof, pt, params, _ = M.case_inputs(c)
        j, plan, dag, profiles = M.run_greedy(dag_spec, prof, pt, params)
        rec = M.serialise_case(c, pt, params, None)
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
