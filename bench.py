#!/usr/bin/env python3
"""Benchmark of the B200 candidate-evaluation path (BASELINE.json metric:
candidate configs evaluated/s; per-window decision latency in ms).

Workload (N = 1 and per GPU count): BASELINE config 5 -- the 6-operator
Llama-2-7B DAG over a synthetic 24 h trace cut into 1440 x 60 s prefill
windows, exhaustive brute-force grid P in {1,2}, R <= 4, B <= 3, i.e.
24^6 = 1.91e8 candidates per window (2.75e11 per step). One step = one pass
of the hot path over the whole batch: per-window prologue, menu build
(predict_op for every (op, P, R, B)), init_configs stability pre-check,
exhaustive compose + SLO mask + lexicographic argmin, per-op fallback,
decode, and plan materialisation (critical path, energy, memory, devices).
At N > 1 every rank enumerates a contiguous slice of every window's
candidate space; the packed keys are min-merged inside the compose kernel
over NVLink peer memory (dist.PeerMerge; --merge nccl: an NCCL MIN
all-reduce after it). Strong scaling: the job is fixed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = ("cfg5: 6-op Llama-2-7B operator DAG, 1440 x 60 s prefill windows of a synthetic "
            "24 h diurnal trace, exhaustive (P in {1,2}, R<=4, B<=3)^6 = 1.91e8 candidates/window")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--merge", choices=("peer", "nccl"), default="peer",
                    help="N>1 key merge: fused into the compose kernel over NVLink peer memory "
                         "(falls back to nccl if peer mapping fails) or an NCCL all-reduce")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload():
    from paper_2511_02248_b200 import model, tables
    from workloads import scenarios
    problem = tables.pack_problem(*scenarios.scenario("cfg5"))
    g = scenarios.GRIDS["cfg5"]
    grid = tables.pack_grid(problem, model.AutoscaleParams(slo=scenarios.SLO["cfg5"]["prefill"]),
                            model.BruteForceBounds(**g))
    tw = scenarios.trace_windows("cfg5")
    win = tables.window_arrays(tw["prefill_qps"], tw["prefill_len"], 0,
                               scenarios.SLO["cfg5"]["prefill"])
    space = 1
    for m in tables.menu_sizes(problem, grid):
        space *= m
    active = int((win.qps > 0).sum())
    return problem, grid, win, space, active


# ---------------------------------------------------------------- CPU arm


CPU_SAMPLE_STEP = 2   # the CPU legs plan every 2nd window (720 of 1440); the GPU arm plans all


def cpu_sample(win):
    idx = np.arange(0, win.n, CPU_SAMPLE_STEP)
    return idx[win.qps[idx] > 0]


def common_config(win, active, space):
    """The `config` both arms print (identical dicts: same workload, same sample)."""
    return {"workload": WORKLOAD, "windows": win.n, "active_windows": active,
            "candidates_per_window": space, "candidates_per_step": active * space,
            "mode": "oracle (exhaustive brute force: every candidate of every window decided)",
            "cpu_sample": f"every {CPU_SAMPLE_STEP}nd window ({len(cpu_sample(win))} of {win.n}): "
                          "the CPU legs (--impl reference, cpu_baseline) plan these per step, the "
                          "GPU arm plans all windows",
            "l2": "flushed between timed GPU steps (256 MiB write outside the events)",
            "workload_choice": "BASELINE config 5 is the throughput config (the 1e8-candidate x "
                               "1440-window sweep sharded over 1/2/4/8 GPUs); config 2 (70B, 1 h "
                               "trace, per-minute windows) is the decision-latency config: "
                               "decision_latency_ms, incl. its batched candidates/s"}


def reference_jobs(win, idx, mode="oracle"):
    return [(mode, float(win.qps[i]), int(win.seq_len[i]), "prefill", float(win.slo[i])) for i in idx]


def cpu_run(problem, grid, win, idx, threads=None):
    """The CPU port (oracle/: the reference's arithmetic restated in C, literal
    enumeration, OpenMP over all host threads) on windows `idx`."""
    from oracle import oracle as orc
    from paper_2511_02248_b200 import abi
    threads = threads or os.cpu_count() or 1
    sub = win.take(idx)
    t = time.perf_counter()
    out = orc.plan_windows(abi.MODE_ORACLE, problem, sub, grid=grid, n_threads=threads)
    return time.perf_counter() - t, threads, out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_grid():
    from workloads import scenarios
    return dict(scenarios.GRIDS["cfg5"])


def reference_arm(args):
    """The reference's own CPU implementation of the path on this host's
    cores: its Python brute_force_autoscale (branch-and-bound + greedy warm
    start, baseline/reference_cpu.py) over one worker process per core, on
    the stated window sample. If the reference package is not installed
    (baseline/_ref), the C port of oracle/ stands in (kind "port")."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(REPO, "baseline"))
    problem, grid, win, space, active = workload()
    idx = cpu_sample(win)
    times = []
    from baseline import reference_cpu as RC
    if RC.available():
        pool = RC.Pool("cfg5", reference_grid())
        jobs = reference_jobs(win, idx)
        for i in range(args.warmup + args.steps):
            wall, _ = pool.run(jobs)
            if i >= args.warmup:
                times.append(wall)
        pool.close()
        kind, cores = "reference", pool.workers
        how = (f"the reference's own brute_force_autoscale (opscaler 0.1.0 from baseline/_ref, "
               f"MAX_ENUMERATION raised), one worker process per core")
        n_win = len(jobs)
    else:
        sub = idx[:: max(1, len(idx) // 72)]
        for i in range(args.warmup + args.steps):
            dt, cores, _ = cpu_run(problem, grid, win, sub)
            if i >= args.warmup:
                times.append(dt)
        kind = "port"
        how = "oracle/ C port (literal enumeration, OpenMP); reference package not installed"
        n_win = len(sub)
    secs = sum(times)
    value = n_win * space * len(times) / secs
    line = {
        "impl": "reference", "metric": "candidate configs evaluated/sec", "value": value,
        "unit": "candidates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / len(times) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": common_config(win, active, space),
        "cpu_baseline": {"value": value, "unit": "candidates/s", "cores": cores, "kind": kind,
                         "sample": f"{n_win} cfg5 prefill windows per step ({how}); semantic "
                                   f"candidates = {space} per window; {cpu_model()}"},
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(problem, grid, win, space, dec):
    """cpu_baseline of the GPU arm (rank 0, after every timed region):
    (1) the reference's own Python brute force over all host cores on the
        stated window sample -- `value`, and its decisions compared with this
        run's GPU decisions (configs, objective, feasibility, latency bits);
    (2) single-process per-window latency of the reference's three planners
        (BASELINE.md CPU plan items 1-2: brute force on cfg5, model level and
        greedy on the 70B cfg2 trace);
    (3) the oracle/ C port (literal enumeration, OpenMP) on the same sample."""
    from baseline import reference_cpu as RC
    from workloads import scenarios
    idx = cpu_sample(win)
    out = {"unit": "candidates/s", "cpu": cpu_model()}
    dt, threads, port = cpu_run(problem, grid, win, idx)
    port_rate = len(idx) * space / dt
    out["port"] = {"value": port_rate, "cores": threads, "seconds": dt,
                   "what": "oracle/ C restatement, literal enumeration of every candidate, OpenMP"}
    if not RC.available():
        out.update(value=port_rate, cores=threads, kind="port",
                   sample=f"{len(idx)} cfg5 prefill windows (every {CPU_SAMPLE_STEP}nd), oracle/ C port")
        return out
    pool = RC.Pool("cfg5", reference_grid())
    jobs = reference_jobs(win, idx)
    pool.run(jobs[: pool.workers])  # worker start-up
    wall, res = pool.run(jobs)
    pool.close()
    ids = problem.ids
    agree = True
    for k, i in enumerate(idx):
        r = res[k][1]
        if isinstance(r, str):
            agree &= int(dec.status[i]) != 0 and not dec.feasible[i]
            continue
        cfgs = tuple(sorted((ids[v], *(int(x) for x in dec.cfg[i, v])) for v in range(len(ids))))
        agree &= (cfgs == r[0] and int(dec.objective[i]) == r[1] and bool(dec.feasible[i]) == r[2]
                  and float(dec.latency[i]).hex() == r[3])
    out.update(value=len(jobs) * space / wall, cores=pool.workers, kind="reference",
               sample=f"{len(jobs)} cfg5 prefill windows (every {CPU_SAMPLE_STEP}nd): the reference's own "
                      f"brute_force_autoscale (branch-and-bound + greedy warm start; semantic "
                      f"candidates = {space} per window), one worker process per core",
               parity_vs_gpu=bool(agree))
    single = {}
    g5 = reference_grid()
    sub = idx[:: max(1, len(idx) // 24)]
    single["brute_force_cfg5"] = RC.per_window_stats(RC.single("cfg5", g5, reference_jobs(win, sub)), space)
    tw = scenarios.trace_windows("cfg2")
    live = np.nonzero(tw["prefill_qps"] > 0)[0][::3]
    jobs2 = lambda mode: [(mode, float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill",
                           scenarios.SLO["cfg2"]["prefill"]) for i in live]
    single["model_level_cfg2_70b"] = RC.per_window_stats(RC.single("cfg2", None, jobs2("model")))
    single["greedy_cfg2_70b"] = RC.per_window_stats(RC.single("cfg2", None, jobs2("operator")))
    out["reference_python_single_process"] = single
    return out


# ---------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.out = index, None, ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- GPU arm


def ours(args):
    import torch

    from paper_2511_02248_b200 import _native, abi, device, tables
    rank, world, local = dist_env()
    # one rank per GPU; OPSC_DIST_BACKEND=gloo (test only) lets several ranks
    # share a GPU to exercise the N>1 path on a 1-GPU box
    backend = os.environ.get("OPSC_DIST_BACKEND", "nccl")
    if world > 1 and backend == "nccl" and torch.cuda.device_count() < world:
        print(f"bench.py: {world} ranks need {world} CUDA devices, {torch.cuda.device_count()} visible",
              file=sys.stderr, flush=True)
        sys.exit(2)
    local = local % max(1, torch.cuda.device_count())
    nccl = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if backend == "nccl":  # communicator setup (ranks, NVLS / P2P transport) logged to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            nccl = ".".join(str(x) for x in torch.cuda.nccl.version())
        dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    problem, grid, win, space, active = workload()
    planner = device.DevicePlanner(problem, win, abi.MODE_ORACLE, grid=grid, device=dev)

    def allreduce(key):
        if world > 1:
            torch.distributed.all_reduce(key, op=torch.distributed.ReduceOp.MIN)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    merge, merge_kind = None, "none" if world == 1 else "nccl all-reduce MIN"
    if world > 1 and args.merge == "peer":
        from paper_2511_02248_b200 import dist as pdist
        try:
            merge = pdist.PeerMerge(win.n, dev)
            # verified once against the NCCL merge before it is used
            planner.step(rank, world, allreduce)
            want = planner.key.clone()
            planner.step(merge=merge)
            merge.check()
            bad = torch.tensor([0 if torch.equal(planner.key, want) else 1], device=dev)
        except Exception as exc:  # noqa: BLE001 -- fall back, consistently on all ranks
            print(f"rank {rank}: peer merge unavailable: {exc}", file=sys.stderr, flush=True)
            bad = torch.tensor([1], device=dev)
        torch.distributed.all_reduce(bad, op=torch.distributed.ReduceOp.MAX)
        if int(bad.item()):
            merge = None
            merge_kind = "nccl all-reduce MIN (peer merge unavailable or mismatched)"
        else:
            merge_kind = "fused: compose CTAs atomicMin into every rank's keys over NVLink peer memory + device barrier"
    for _ in range(args.warmup):
        planner.step(rank, world, allreduce, merge=merge)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches0 = planner.launches
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 (126 MB) flushed between timed steps, outside the events
            ev[i][0].record()
            planner.step(rank, world, allreduce, compose_events=cev[i], merge=merge)
            ev[i][1].record()
        barrier()
    launches = planner.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    comp_ms = [a.elapsed_time(b) for a, b in cev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(tot.item())
    cands_step = active * space
    value = cands_step * args.steps / (total_ms * 1e-3)

    # parity of this very run against the CPU oracle on a few windows
    dec = planner.decisions()
    parity = None
    if rank == 0:
        from oracle import oracle as orc
        idx = np.array([0, 719, 1439])
        ref = orc.plan_windows(abi.MODE_ORACLE, problem, win.take(idx), grid=grid)
        parity = all(getattr(dec, f)[idx].tobytes() == getattr(ref, f).tobytes()
                     for f in ("key", "cfg", "latency", "energy", "memory", "devices"))
    # summation-order certificate over every window of this run (outside the
    # timed region): argmin at slo -/+ 64 ulps must agree, else the decision
    # could depend on the reference's frozenset-ordered leaf sum
    certificate = None
    if rank == 0:
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        planner.certify()
        c1.record()
        c1.synchronize()
        st = planner.out_t["status"].cpu().numpy().view(np.uint32)
        certificate = {"windows": int(win.n), "band_ulps": abi.CERTIFY_BAND_ULPS,
                       "order_sensitive_windows": int(((st & abi.W_ORDER_SENSITIVE) != 0).sum()),
                       "ms": c0.elapsed_time(c1),
                       "what": "OPSC_W_ORDER_SENSITIVE: argmin(lat <= slo - band) != argmin(lat <= slo + band)"}

    # roofline of the dominant kernel (compose_argmin)
    peak = device.fp64_peak()
    comp_avg = sum(comp_ms) / len(comp_ms) * 1e-3
    my_cands = cands_step / world
    achieved = 2.0 * my_cands / comp_avg  # DADD + DSETP per composed candidate
    n_ops = problem.n_ops
    traffic = None
    tp = os.path.join(REPO, "profiles", "compose_ncu_summary.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    # e2e through the C-ABI host-buffer call (pinned host windows in, decisions out)
    e2e = None
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hwin = tables.WindowArrays(*(pin(getattr(win, k)) for k in ("qps", "seq_len", "phase", "slo", "eps")))
    hout = tables.DecisionArrays(win.n, n_ops)
    for f in tables.DecisionArrays.FIELDS:
        setattr(hout, f, pin(getattr(hout, f)))
    bi = sum(getattr(hwin, k).nbytes for k in ("qps", "seq_len", "phase", "slo", "eps"))
    if world > 1:
        # N ranks: host windows in, this rank's candidate shard, NCCL MIN merge,
        # decode + materialise, decisions back to host on every rank
        from paper_2511_02248_b200 import dist as pdist
        for _ in range(args.warmup):
            pdist.plan_windows_host_sharded(planner, hwin, hout, merge=merge)
        t, wall = [], []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            planner.load_windows(hwin)  # H2D (pinned, async)
            if merge is not None:
                planner.step(merge=merge)
            else:
                pdist.plan_windows_sharded(planner)
            planner.fetch(hout, sync=False)  # D2H (pinned, async)
            e1.record()
            e1.synchronize()
            wall.append(time.perf_counter() - t0)
            t.append(e0.elapsed_time(e1) * 1e-3)
        tt = torch.tensor([sum(t), sum(wall)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": cands_step * len(t) / float(tt[0].item()), "unit": "candidates/s",
               "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(hout.nbytes()),
               "api": "dist.plan_windows_host_sharded's steps (host buffers, shard per rank, key merge)",
               "timing": "CUDA events on the rank's stream around H2D .. D2H, max over ranks",
               "wall_value": cands_step * len(t) / float(tt[1].item()),
               "parity_vs_device_path": bool(all(
                   getattr(hout, f).tobytes() == getattr(dec, f).tobytes()
                   for f in ("key", "cfg", "latency", "energy")))}
    if world == 1:
        ctx = _native.Context(device=local, max_windows=win.n)
        for _ in range(args.warmup):
            ctx.plan_windows(abi.MODE_ORACLE, problem, hwin, grid=grid, out=hout)
        t, wall = [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            ctx.plan_windows(abi.MODE_ORACLE, problem, hwin, grid=grid, out=hout)
            wall.append(time.perf_counter() - t0)
            t.append(ctx.last_ms() * 1e-3)
        e2e_launches = ctx.last_launches()
        ctx.close()
        bi = sum(getattr(hwin, k).nbytes for k in ("qps", "seq_len", "phase", "slo", "eps"))
        e2e = {"value": cands_step * len(t) / sum(t), "unit": "candidates/s",
               "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(hout.nbytes()),
               "api": "opsc_plan_windows_host (C ABI, host buffers)",
               "timing": "CUDA events on the context stream around the call's first H2D .. last D2H "
                         "(opsc_ctx_last_ms)",
               "wall_value": cands_step * len(wall) / sum(wall),
               "launches_per_step": e2e_launches,
               "parity_vs_device_path": bool(all(
                   getattr(hout, f).tobytes() == getattr(dec, f).tobytes()
                   for f in ("key", "cfg", "latency", "energy")))}

    # per-window decision latency on the 70B DAG (cfg2), W = 1
    latency = None
    if rank == 0 and not args.no_latency:
        latency = decision_latency(dev)
        latency["trace_pipeline"] = trace_pipeline(dev)
        latency["capacity_8gpu"] = capacity_8gpu(dev)
        latency["multimodal_cfg3"] = multimodal_batched(dev)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # after every timed region; other ranks wait
        cpu = cpu_baseline(problem, grid, win, space, dec)

    if rank == 0:
        line = {
            "metric": "candidate configs evaluated/sec", "value": value, "unit": "candidates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": common_config(win, active, space),
            "run": {"parallelism": f"candidate-range shards x{world}" if world > 1 else "single GPU",
                    "merge": merge_kind, "dist_backend": backend if world > 1 else None,
                    "nccl_version": nccl},
            "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel": "compose_kernel (opsc_compose_argmin)",
                         "algorithmic_ops_per_candidate": 2,
                         "peak_source": "live DADD microbenchmark (opsc_fp64_peak); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "survey_n_ops_per_candidate": n_ops,
                         "survey_frac": n_ops * my_cands / comp_avg / peak,
                         "kernel_ms": comp_avg * 1e3,
                         "kernel_share_of_step": comp_avg * 1e3 / (sum(step_ms) / len(step_ms))},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "decision_latency_ms": latency,
            "parity_vs_oracle": parity,
            "order_certificate": certificate,
        }
        print(json.dumps(line), flush=True)
    if merge is not None:
        merge.check()
        merge.close()
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def decision_latency(dev):
    """Window stats resident on device -> decoded decision, one window at a
    time, for the 10-op Llama-2-70B DAG (cfg2): exhaustive oracle over
    (P in {2,4}, R<=3, B=1)^10 = 6.0e7 candidates, the model-level grid and
    greedy. `feasible_windows` counts the windows whose decision is a feasible
    winner (the rest are infeasible-SLO fallbacks or NoStableConfig)."""
    import torch

    from paper_2511_02248_b200 import abi, device, model, tables
    from workloads import scenarios
    problem = tables.pack_problem(*scenarios.scenario("cfg2"))
    g = scenarios.GRIDS["cfg2"]
    tw = scenarios.trace_windows("cfg2")
    out = {}
    for mode, name in ((abi.MODE_ORACLE, "oracle_6e7_candidates"), (abi.MODE_MODEL, "model_level"),
                       (abi.MODE_OPERATOR, "operator_greedy")):
        samples, eager = [], []
        batch_ms = 0.0
        n_feas = n_nostable = 0
        for phase in ("prefill", "decode"):
            slo = scenarios.SLO["cfg2"][phase]
            params = model.AutoscaleParams(slo=slo)
            grid = tables.pack_grid(problem, params, model.BruteForceBounds(**g))
            spec = tables.pack_model(problem, params)
            gspec = tables.pack_greedy(problem, params)
            qs, ls = tw[phase + "_qps"], tw[phase + "_len"]
            # whole trace in one batch
            allw = tables.window_arrays(qs, ls, tables.PHASE_INDEX[phase], slo)
            pb = device.DevicePlanner(problem, allw, mode, grid=grid, model=spec, greedy=gspec,
                                      device=dev)
            pb.step()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record()
            pb.step()
            b1.record()
            b1.synchronize()
            batch_ms += b0.elapsed_time(b1)
            live = torch.from_numpy(np.asarray(qs > 0)).to(dev)
            n_feas += int((pb.out_t["feasible"].bool() & live).sum())
            nst = abi.W_NO_STABLE_BOUNDS | abi.W_NO_STABLE_PARAMS | abi.W_NO_STABLE_MODEL | abi.W_NO_STABLE_INIT
            n_nostable += int(((pb.out_t["status"] & nst) != 0).sum())
            one = tables.window_arrays(qs[:1], ls[:1], tables.PHASE_INDEX[phase], slo)
            p = device.DevicePlanner(problem, one, mode, grid=grid, model=spec, greedy=gspec,
                                     device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            graph = p.capture()  # the per-window pipeline as one CUDA graph launch
            for i in range(len(qs)):
                if not qs[i] > 0:
                    continue
                p.win_t["qps"].fill_(float(qs[i]))
                p.win_t["seq_len"].fill_(int(ls[i]))
                torch.cuda.synchronize(dev)
                e0.record()
                p.step()
                e1.record()
                e1.synchronize()
                eager.append(e0.elapsed_time(e1))
                torch.cuda.synchronize(dev)
                e0.record()
                graph.replay()
                e1.record()
                e1.synchronize()
                samples.append(e0.elapsed_time(e1))
        samples.sort()
        eager.sort()
        out[name] = {"median": statistics.median(samples),
                     "p99": samples[min(len(samples) - 1, int(0.99 * len(samples)))],
                     "windows": len(samples),
                     "launch": "CUDA graph replay of the whole per-window pipeline",
                     "eager_median": statistics.median(eager),
                     "eager_p99": eager[min(len(eager) - 1, int(0.99 * len(eager)))],
                     "batched_ms_per_window": batch_ms / max(1, len(samples)),
                     "feasible_windows": n_feas, "no_stable_config_windows": n_nostable}
        if mode == abi.MODE_ORACLE:  # cfg2 throughput: whole trace per launch set, 6^10 candidates per window
            cpw = 1
            for v in range(problem.n_ops):
                cpw *= grid.menu_off[v + 1] - grid.menu_off[v]
            out[name]["batched_candidates_per_s"] = cpw / (out[name]["batched_ms_per_window"] * 1e-3)
    out["dag"] = "cfg2 Llama-2-70B 10-op chain, 60 x 60 s windows x {prefill, decode}, W = 1"
    return out


def multimodal_batched(dev):
    """Config 3: the 12-op multimodal DAG (vision branch + text embed merging
    into the LLM stack, heavy-tailed lengths) over its whole trace, both
    phases, one launch set per phase: exhaustive (P in {1,2}, R<=3, B=1)^12 =
    2.2e9 candidates per window, model level and greedy."""
    import torch

    from paper_2511_02248_b200 import abi, device, model, tables
    from workloads import scenarios
    problem = tables.pack_problem(*scenarios.scenario("cfg3"))
    g = scenarios.GRIDS["cfg3"]
    tw = scenarios.trace_windows("cfg3")
    out = {"dag": "cfg3 multimodal 12-op DAG (two sources), whole trace x {prefill, decode}, one launch set per phase"}
    for mode, name in ((abi.MODE_ORACLE, "oracle"), (abi.MODE_MODEL, "model_level"),
                       (abi.MODE_OPERATOR, "operator_greedy")):
        ms, n_win, cands = 0.0, 0, 0
        for phase in ("prefill", "decode"):
            slo = scenarios.SLO["cfg3"][phase]
            params = model.AutoscaleParams(slo=slo)
            grid = tables.pack_grid(problem, params, model.BruteForceBounds(**g))
            qs, ls = tw[phase + "_qps"], tw[phase + "_len"]
            allw = tables.window_arrays(qs, ls, tables.PHASE_INDEX[phase], slo)
            pb = device.DevicePlanner(problem, allw, mode, grid=grid, model=tables.pack_model(problem, params),
                                      greedy=tables.pack_greedy(problem, params), device=dev)
            pb.step()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pb.step()
            e1.record()
            e1.synchronize()
            ms += e0.elapsed_time(e1)
            active = int((qs > 0).sum())
            n_win += active
            cpw = 1
            for v in range(problem.n_ops):
                cpw *= grid.menu_off[v + 1] - grid.menu_off[v]
            cands += cpw * active
        out[name] = {"ms": ms, "windows": n_win, "ms_per_window": ms / max(1, n_win)}
        if mode == abi.MODE_ORACLE:
            out[name]["candidates"] = cands
            out[name]["candidates_per_s"] = cands / (ms * 1e-3)
    return out


def capacity_8gpu(dev):
    """Config 4 (an extension without reference semantics):
    per window, the largest arrival rate whose exhaustive min-objective
    decision fits 8 x 80 GB devices -- batched k-ary bisection, each round one
    planning launch set over windows x 32 rates."""
    import torch

    from paper_2511_02248_b200 import capacity, model
    from workloads import scenarios
    dag, prof = scenarios.scenario("cfg1")
    tw = scenarios.trace_windows("cfg2")
    idx = np.linspace(0, 59, 8).round().astype(int)
    pts = [model.WorkloadPoint(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill") for i in idx]
    params = model.AutoscaleParams(slo=scenarios.SLO["cfg1"]["prefill"])
    bounds = model.BruteForceBounds(**scenarios.GRIDS["cfg1"])
    capacity.max_qps_under_budget(dag, prof, pts[:1], params, bounds=bounds, max_rounds=1)  # warm-up
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    res = capacity.max_qps_under_budget(dag, prof, pts, params, bounds=bounds, budget=8, mem_cap=80e9,
                                        fan=32, rel_tol=1e-6)
    dt = time.perf_counter() - t
    return {"dag": "cfg1 7B 6-op, exhaustive 12^6 grid, 8 windows of the cfg2 trace (prefill)",
            "budget": "8 x 80 GB, default-stream devices_used", "ms": dt * 1e3, "rounds": res.rounds,
            "plans_evaluated": res.evaluated, "candidates_composed": res.evaluated * 12 ** 6,
            "max_qps": [float(x) for x in res.qps], "devices": [int(x) for x in res.devices]}


def trace_pipeline(dev):
    """Whole 1 h cfg2 trace (records resident in HBM) -> per-window decisions
    for both phases: GPU windowize + planner + materialise, CUDA events
    around the call (includes the host's launch gaps)."""
    import torch

    from paper_2511_02248_b200 import model, pipeline, workload
    from workloads import scenarios
    spec = scenarios.TRACES["cfg2"]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    arr = torch.tensor([r.arrival_time for r in recs], dtype=torch.float64, device=dev)
    li = torch.tensor([r.input_len for r in recs], dtype=torch.int32, device=dev)
    lo = torch.tensor([r.output_len for r in recs], dtype=torch.int32, device=dev)
    dag, prof = scenarios.scenario("cfg2")
    params = {ph: model.AutoscaleParams(slo=scenarios.SLO["cfg2"][ph]) for ph in ("prefill", "decode")}
    out = {"trace": "cfg2 1 h burst trace", "records": len(recs)}
    for mode in ("operator", "model", "oracle"):
        bounds = model.BruteForceBounds(**scenarios.GRIDS["cfg2"]) if mode == "oracle" else None
        tp = pipeline.TracePlanner(dag, prof, params, mode, bounds, device_=dev)
        tp.run(arr, li, lo)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record()
            res = tp.run(arr, li, lo)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[mode + "_ms"] = statistics.median(ts)
        out["windows"] = res["prefill"].W
    return out


def spawn(args):
    """`--gpus N` (N > 1) outside torchrun: re-exec this command under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous). The
    GPU arm refuses to start when fewer than N devices are visible instead of
    silently time-sharing one."""
    if args.impl == "ours" and os.environ.get("OPSC_DIST_BACKEND", "nccl") == "nccl":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {n} visible",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1 and args.impl == "ours":
            spawn(args)
    elif int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}",
              file=sys.stderr, flush=True)
        sys.exit(2)
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
