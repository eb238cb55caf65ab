"""Per-window (W=1) pipelines for ncu launch timing (dev tool)."""
import sys
import torch
from paper_2511_02248_b200 import abi, device, model, scenarios, tables

prob = tables.pack_problem(*scenarios.scenario("cfg2"))
tw = scenarios.trace_windows("cfg2")
params = model.AutoscaleParams(slo=2.0)
mode = {"model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR, "oracle": abi.MODE_ORACLE}[sys.argv[1]]
i = int(sys.argv[2]) if len(sys.argv) > 2 else 7
win = tables.window_arrays(tw["prefill_qps"][i:i + 1], tw["prefill_len"][i:i + 1], 0, 2.0)
p = device.DevicePlanner(prob, win, mode, grid=tables.pack_grid(prob, params, model.BruteForceBounds(**scenarios.GRIDS["cfg2"])),
                         model=tables.pack_model(prob, params), greedy=tables.pack_greedy(prob, params))
for _ in range(3):
    p.step()
torch.cuda.synchronize()
d = p.decisions()
print("cfg", d.cfg[0].tolist(), "lat", d.latency[0], "trace_len", d.trace_len[0] if p.trace_cap else None)
