"""Multi-GPU planning: candidate-range sharding + one MIN all-reduce.

Every window's candidate space [0, prod m_i) is split into contiguous
shards, one per rank (opsc_compose_argmin's `shard / n_shards`). Each rank
min-reduces its shard to a packed key (objective << 40 | lexicographic
index); since the key embeds the global lexicographic index, the MIN
all-reduce over ranks (NCCL over NVLink on GPUs, gloo in the CPU tests)
returns exactly the single-GPU decision for any world size. Menus are cheap
(~1 us per window) and are rebuilt on every rank, so the all-reduce of
[W] int64 keys is the only data-path exchange.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import abi


def merge_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """In-place MIN all-reduce of per-window packed keys (int64)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    return keys


def rank_shard(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def plan_windows_sharded(planner, group=None):
    """Run one DevicePlanner step with this rank's shard and the NCCL merge;
    every rank ends with the full decisions of every window."""
    rank, world = rank_shard(group)
    planner.step(rank, world, allreduce=lambda k: merge_keys(k, group))
    return planner


def plan_windows_host_sharded(planner, host_windows, host_out, group=None, merge=None):
    """Host buffers in, decisions out, on N ranks: H2D of the window SoA,
    this rank's candidate shard, the MIN merge (fused into the compose
    kernel over peer memory with `merge`, else an NCCL all-reduce), decode
    + materialise, D2H. `host_out` (tables.DecisionArrays) ends with the
    full decisions on every rank."""
    planner.load_windows(host_windows)
    if merge is not None:
        planner.step(merge=merge)
    else:
        plan_windows_sharded(planner, group)
    return planner.fetch(host_out)


def infeasible_keys(n, device="cpu"):
    return torch.full((n,), abi.KEY_INFEASIBLE, dtype=torch.int64, device=device)


class PeerMerge:
    """The MIN merge fused into the compose kernel over NVLink peer memory.

    Every rank owns one CUDA-IPC-shared allocation: two [W] int64 key
    buffers and a [world] uint32 arrival-flag array. The compose kernel
    (opsc_compose_argmin_peers) atomicMin's each CTA's key straight into the
    current key buffer of EVERY rank, so the merge overlaps the enumeration
    tile by tile; one device flag barrier (opsc_peer_barrier) then orders all
    ranks' atomics before decode. The buffer for step s+1 is reset before
    the barrier of step s, so no rank can write into a buffer a peer has not
    yet reset (double buffering, one barrier per step).
    """

    def __init__(self, n_windows, device, group=None, timeout_ms=10_000):
        import ctypes as C

        from . import _native
        self.C, self.L = C, _native.load()
        self.rank, self.world = rank_shard(group)
        if self.world > abi.MAX_PEERS:
            raise ValueError(f"peer merge supports up to {abi.MAX_PEERS} ranks (one node)")
        self.dev = torch.device(device)
        if self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        torch.cuda.set_device(self.dev)
        self.W, self.timeout_ms, self.group = int(n_windows), int(timeout_ms), group
        self.flag_off = 2 * self.W * 8
        nbytes = self.flag_off + 4 * abi.MAX_PEERS
        ptr, handle = C.c_void_p(), (C.c_ubyte * abi.IPC_HANDLE_BYTES)()
        rc = self.L.opsc_ipc_alloc(nbytes, C.cast(C.byref(ptr), C.c_void_p), C.cast(handle, C.c_void_p))
        self.local, self.opened = (ptr.value if rc == abi.OK else None), []
        handles = self._agree(bytes(handle) if rc == abi.OK else None, "ipc_alloc")
        self.base = []
        failure = None
        for r, h in enumerate(handles):
            if r == self.rank:
                self.base.append(self.local)
                continue
            p = C.c_void_p()
            hb = (C.c_ubyte * abi.IPC_HANDLE_BYTES).from_buffer_copy(h)
            rc = self.L.opsc_ipc_open(C.cast(hb, C.c_void_p), C.cast(C.byref(p), C.c_void_p))
            if rc != abi.OK:
                failure = failure or f"ipc_open of rank {r}: {self.L.opsc_status_string(rc).decode()}"
                continue
            self.base.append(p.value)
            self.opened.append(p.value)
        self._agree(failure is None or None, failure or "")
        self.flags = (C.c_void_p * self.world)(*[b + self.flag_off for b in self.base])
        self.err = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.epoch, self.buf = 0, 0
        s = self._s()
        for b in (0, 1):
            _native.check(self.L.opsc_fill_keys(self.key_ptr(b), self.W, s), "fill_keys")
        self.barrier()
        self.check()

    def _agree(self, mine, what):
        """All-gather this rank's value; every rank raises if any rank
        failed (None), so no rank is left waiting in a later collective."""
        if self.world > 1:
            vals = [None] * self.world
            dist.all_gather_object(vals, mine, group=self.group)
        else:
            vals = [mine]
        if any(v is None for v in vals):
            self.close(collective=False)
            raise RuntimeError(f"peer merge setup failed on rank(s) "
                               f"{[i for i, v in enumerate(vals) if v is None]}: {what}")
        return vals

    def _s(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def key_ptr(self, b, r=None):
        return self.base[self.rank if r is None else r] + b * self.W * 8

    def key_ptrs(self, b):
        return (self.C.c_void_p * self.world)(*[self.key_ptr(b, r) for r in range(self.world)])

    def barrier(self):
        from . import _native
        self.epoch += 1
        _native.check(self.L.opsc_peer_barrier(self.flags, self.rank, self.world, self.epoch, self.timeout_ms,
                                               self.err.data_ptr(), self._s()), "peer_barrier")

    def check(self):
        """Raise if any barrier timed out (syncs the stream)."""
        if int(self.err.item()):
            raise RuntimeError("peer barrier timed out: a rank did not arrive")

    def step(self, planner, compose_events=None):
        """One merged step of a DevicePlanner (oracle mode): compose with
        fused peer atomics, reset the next buffer, barrier, decode."""
        from . import _native
        r, L, s = _native.ref, self.L, self._s()
        cur = self.buf
        planner._init(reset_key=False)
        planner.menus()
        if compose_events:
            compose_events[0].record()
        planner._ck(L.opsc_compose_argmin_peers(r(planner.problem.table), r(planner.grid), planner.win,
                                                planner.menu.data_ptr(), self.rank, self.world,
                                                self.key_ptrs(cur), self.world, s), "compose_argmin_peers")
        if compose_events:
            compose_events[1].record()
        planner._ck(L.opsc_fill_keys(self.key_ptr(1 - cur), self.W, s), "fill_keys")
        self.barrier()
        planner._ck(L.opsc_copy_keys(planner.key.data_ptr(), self.key_ptr(cur), self.W, s), "copy_keys")
        planner.finish()
        self.buf = 1 - cur

    def close(self, collective=True):
        torch.cuda.synchronize(self.dev)
        if collective and self.world > 1:
            dist.barrier(group=self.group)
        for p in getattr(self, "opened", []):
            self.L.opsc_ipc_close(p)
        self.opened = []
        if collective and self.world > 1:
            dist.barrier(group=self.group)
        if self.local:
            self.L.opsc_ipc_free(self.local)
            self.local = None
