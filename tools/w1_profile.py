"""Per-window (W=1) pipelines for ncu launch timing / source profiles (dev tool).

    python tools/w1_profile.py {model,operator,oracle} [window] [prefill|decode]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import abi, device, model, tables  # noqa: E402
from workloads import scenarios  # noqa: E402

prob = tables.pack_problem(*scenarios.scenario("cfg2"))
tw = scenarios.trace_windows("cfg2")
mode = {"model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR, "oracle": abi.MODE_ORACLE}[sys.argv[1]]
i = int(sys.argv[2]) if len(sys.argv) > 2 else 7
ph = sys.argv[3] if len(sys.argv) > 3 else "prefill"
slo = scenarios.SLO["cfg2"][ph]
params = model.AutoscaleParams(slo=slo)
win = tables.window_arrays(tw[ph + "_qps"][i:i + 1], tw[ph + "_len"][i:i + 1], tables.PHASE_INDEX[ph], slo)
p = device.DevicePlanner(prob, win, mode, grid=tables.pack_grid(prob, params, model.BruteForceBounds(**scenarios.GRIDS["cfg2"])),
                         model=tables.pack_model(prob, params), greedy=tables.pack_greedy(prob, params))
for _ in range(3):
    p.step()
torch.cuda.synchronize()
d = p.decisions()
print("cfg", d.cfg[0].tolist(), "lat", d.latency[0], "trace_len", d.trace_len[0] if p.trace_cap else None)
