"""Dev tool: windowize alone (cfg2 1 h trace, records resident) and the
whole trace pipeline, CUDA-event medians (one line)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_02248_b200 import workload  # noqa: E402
from workloads import scenarios  # noqa: E402

dev = torch.device("cuda")
spec = scenarios.TRACES["cfg2"]
recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
arr = torch.tensor([r.arrival_time for r in recs], dtype=torch.float64, device=dev)
li = torch.tensor([r.input_len for r in recs], dtype=torch.int32, device=dev)
lo = torch.tensor([r.output_len for r in recs], dtype=torch.int32, device=dev)
ts = []
for i in range(25):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    workload.windowize_device(arr, li, lo, spec["window_len"], spec["quantile"], dev)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
tp = bench.trace_pipeline(dev)
print(f"windowize {statistics.median(ts[5:]):.4f} ms | pipeline operator {tp['operator_ms']:.4f} model {tp['model_ms']:.4f} oracle {tp['oracle_ms']:.4f} ms")
