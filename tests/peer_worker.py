"""Worker for tests/test_gpu_peer.py: N ranks (sharing one GPU under the
test's gloo group, or one GPU each) plan cfg5 windows with the merge fused
into the compose kernel over IPC peer memory, for several steps, and check
every rank's decisions against a single-rank plan. Exit 0 on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02248_b200 import abi, device, dist as pdist, model, tables  # noqa: E402
from workloads import scenarios  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(os.environ.get("OPSC_DIST_BACKEND", "gloo"))
    dev = torch.device("cuda", local)
    prob = tables.pack_problem(*scenarios.scenario("cfg5"))
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=0.5), model.BruteForceBounds(**scenarios.GRIDS["cfg5"]))
    tw = scenarios.trace_windows("cfg5")
    idx = np.arange(0, 1440, 15)
    qps = tw["prefill_qps"][idx].copy()
    qps[3] = 0.0  # an idle window: no atomics, key stays +inf
    win = tables.window_arrays(qps, tw["prefill_len"][idx], 0, 0.5)
    ref = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid, device=dev)
    ref.step()
    want = ref.decisions()
    planner = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid, device=dev)
    merge = pdist.PeerMerge(win.n, dev)
    ok = True
    for step in range(4):
        planner.step(merge=merge)
        merge.check()
        got = planner.decisions()
        for f in ("key", "cfg", "feasible", "status", "latency", "objective", "energy", "memory", "devices"):
            if getattr(got, f).tobytes() != getattr(want, f).tobytes():
                print(f"rank {rank} step {step}: {f} differs", flush=True)
                ok = False
    merge.close()
    flag = torch.tensor([0 if ok else 1], dtype=torch.int32,
                        device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    print(f"rank {rank}/{world}: {'ok' if int(flag) == 0 else 'FAILED'}", flush=True)
    sys.exit(0 if int(flag) == 0 else 1)


if __name__ == "__main__":
    main()
