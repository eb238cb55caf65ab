"""W=1 decision latency (CUDA-graph replay) over cfg2 windows for one mode (dev tool).

    python tools/w1_latency.py {oracle,model,operator} [n_windows]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import abi, device, model, tables  # noqa: E402
from workloads import scenarios  # noqa: E402

mode = {"model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR, "oracle": abi.MODE_ORACLE}[sys.argv[1]]
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if os.environ.get("OPSC_MODEL_TABLE_POINTS"):  # dev override of the small-batch table threshold
    device.DevicePlanner.MODEL_TABLE_POINTS = int(os.environ["OPSC_MODEL_TABLE_POINTS"])
prob = tables.pack_problem(*scenarios.scenario("cfg2"))
tw = scenarios.trace_windows("cfg2")
out = []
for ph in ("prefill", "decode"):
    slo = scenarios.SLO["cfg2"][ph]
    params = model.AutoscaleParams(slo=slo)
    qs, ls = tw[ph + "_qps"], tw[ph + "_len"]
    one = tables.window_arrays(qs[:1], ls[:1], tables.PHASE_INDEX[ph], slo)
    p = device.DevicePlanner(prob, one, mode, grid=tables.pack_grid(prob, params, model.BruteForceBounds(**scenarios.GRIDS["cfg2"])),
                             model=tables.pack_model(prob, params), greedy=tables.pack_greedy(prob, params))
    g = p.capture()
    g.replay()  # warm-up: the first replay uploads the graph
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(nw):
        p.win_t["qps"].fill_(float(qs[i]))
        p.win_t["seq_len"].fill_(int(ls[i]))
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
        if os.environ.get("W1_DETAIL"):
            tl = int(p.trace_len[0].item()) if p.trace_cap else -1
            print(f"  {ph} w{i}: {out[-1]:.4f} ms trace_len {tl} status {int(p.out_t['status'][0].item()):#x}")
srt = sorted(out)
print(f"{sys.argv[1]} IL={os.environ.get('OPSC_COMPOSE_IL', 'auto')}: median {statistics.median(out):.4f} ms, "
      f"p99 {srt[min(len(srt) - 1, int(0.99 * len(srt)))]:.4f} ms, max {srt[-1]:.4f} ms over {len(out)} windows")
