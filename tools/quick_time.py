"""Quick device timing of the exhaustive pipeline (dev tool): cfg5 (default) or cfg2.

    python tools/quick_time.py [cfg5|cfg2]
"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_02248_b200 import _native, abi, model, tables
from workloads import scenarios

nat = _native
L = nat.load()
CFG = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
prob = tables.pack_problem(*scenarios.scenario(CFG))
g = scenarios.GRIDS[CFG]
grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**g))
tw = scenarios.trace_windows(CFG)
win = tables.window_arrays(tw["prefill_qps"], tw["prefill_len"], 0, scenarios.SLO[CFG]["prefill"])
dev = torch.device("cuda:0")
t = {k: torch.from_numpy(np.array(getattr(win, k))).to(dev) for k in ("qps", "seq_len", "phase", "slo", "eps")}
dw = abi.OpscWindows(); dw.n = win.n
for k in t: setattr(dw, k, t[k].data_ptr())
E = grid.menu_off[prob.n_ops]
mw = torch.empty((win.n, E), dtype=torch.float64, device=dev)
st = torch.zeros(win.n, dtype=torch.int32, device=dev)
key = torch.empty(win.n, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream().cuda_stream
def step():
    nat.check(L.opsc_menu_build(nat.ref(prob.table), nat.ref(grid), dw, mw.data_ptr(), st.data_ptr(), s), "m")
    nat.check(L.opsc_fill_keys(key.data_ptr(), win.n, s), "f")
    nat.check(L.opsc_compose_argmin(nat.ref(prob.table), nat.ref(grid), dw, mw.data_ptr(), 0, 1, key.data_ptr(), s), "c")
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(5): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
cands = win.n * int(np.prod([grid.menu_off[v + 1] - grid.menu_off[v] for v in range(prob.n_ops)]))
print(f"{CFG} step {ms:.3f} ms  candidates {cands:.3e}  rate {cands/ms*1e3:.3e}/s")
ms2 = ctypes_ms = None
import ctypes as C
f = C.c_float(); ops = C.c_double()
nat.check(L.opsc_fp64_peak(20000, C.cast(C.byref(f), C.c_void_p), C.cast(C.byref(ops), C.c_void_p), s), "peak")
print(f"fp64 DADD peak: {ops.value/f.value*1e3:.3e} op/s ({f.value:.2f} ms)")
k = key.cpu().numpy()
print("feasible windows", (k != abi.KEY_INFEASIBLE).sum())
for kind, name in ((1, "literal DADD+DSETP+SEL"), (2, "threshold DSETP+SEL")):
    nat.check(L.opsc_candidate_probe(kind, 20000, C.cast(C.byref(f), C.c_void_p), C.cast(C.byref(ops), C.c_void_p), s), "probe")
    print(f"probe {name}: {ops.value/f.value*1e3:.3e} candidates/s ({f.value:.2f} ms)")
