"""One pass of the trace -> decisions -> placement pipeline for ncu (dev
tool): cfg2 (70B DAG) 1 h trace, windowize on device, greedy operator-level
planning for both phases, shared placement of the prefill plans.

    ncu --set full -o gpurun_out/pipeline python tools/profile_pipeline.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import model, pipeline, placement, workload  # noqa: E402
from workloads import scenarios  # noqa: E402


def main():
    spec = scenarios.TRACES["cfg2"]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    arr = np.array([r.arrival_time for r in recs])
    li = np.array([r.input_len for r in recs])
    lo = np.array([r.output_len for r in recs])
    dag, prof = scenarios.scenario("cfg2")
    params = {ph: model.AutoscaleParams(slo=scenarios.SLO["cfg2"][ph]) for ph in ("prefill", "decode")}
    mode = sys.argv[1] if len(sys.argv) > 1 else "operator"
    tp = pipeline.TracePlanner(dag, prof, params, mode)
    res = tp.run(arr, li, lo)
    pre = res["prefill"]
    dec = pre.decisions()
    fleet = placement.SharedFleet(model.make_fleet(1024, 180e9), 2.0, model.InterferenceParams(0.5, 1.0),
                                  model.EnergyParams())
    from paper_2511_02248_b200 import tables
    win = tables.WindowArrays(*(pre.win_t[k].cpu().numpy() for k in ("qps", "seq_len", "phase", "slo", "eps")))
    placement.place_windows(tp.problem, win, dec.cfg, dec.feasible, fleet, 1)
    torch.cuda.synchronize()
    print("windows", win.n, "feasible", int(dec.feasible.sum()))


if __name__ == "__main__":
    main()
