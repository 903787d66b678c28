"""Cache Manager / Communication Group Pool and the process topology.

The reference models the pool as a grow-only set of (tp, dp) layouts whose
first use costs `comm_init_cost` (CommGroupPool, tpshift/switchcost.py:76-104).
On B200 a "communicator" is a table of NVLink-peer device pointers plus the
device counters of the one-shot allreduce: created lazily per layout, cached
for the life of the worker, never torn down (idle tables cost a few MB).

World topology: one process per GPU (torchrun, NCCL/gloo only for host-side
handle exchange) or a *virtual* world where one process drives every rank on
one device (single-GPU tests and microbenchmarks). Peer pointers come from
CUDA IPC across processes and are plain device pointers inside a process.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _native as nat
from .executor import GroupComm


@dataclass
class World:
    gpus: int                       # ranks of the node
    local_ranks: list[int]          # ranks this process drives
    devices: dict[int, torch.device]
    distributed: bool = False       # torch.distributed initialised (one process per GPU)
    _ipc_cache: dict = field(default_factory=dict)

    @classmethod
    def virtual(cls, gpus: int, device="cuda:0") -> "World":
        d = torch.device(device)
        return cls(gpus=gpus, local_ranks=list(range(gpus)), devices={r: d for r in range(gpus)})

    @classmethod
    def from_env(cls) -> "World":
        """One process per GPU under torchrun (RANK/LOCAL_RANK/WORLD_SIZE)."""
        import os

        import torch.distributed as dist
        n = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        # TPS_SHARE_DEVICE=1: every rank's process on cuda:0 (the IPC/peer-counter path of a
        # multi-GPU node exercised on one device; the kernels time-slice between processes)
        d = torch.device("cuda:0" if os.environ.get("TPS_SHARE_DEVICE") == "1" else f"cuda:{local}")
        torch.cuda.set_device(d)
        if n > 1 and not dist.is_initialized():
            dist.init_process_group(backend="gloo")
        return cls(gpus=n, local_ranks=[rank], devices={rank: d}, distributed=n > 1)

    @property
    def is_virtual(self) -> bool:
        return len(self.local_ranks) > 1

    def allgather(self, obj):
        if not self.distributed:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.gpus
        dist.all_gather_object(out, obj)
        return out

    def barrier(self) -> None:
        if self.distributed:
            import torch.distributed as dist
            dist.barrier()

    # ---- peer pointers -------------------------------------------------
    def share(self, tensors: dict[int, dict[str, torch.Tensor]]) -> dict[int, dict[str, int]]:
        """Make {rank: {name: tensor}} of every rank addressable here: {rank: {name: ptr}}."""
        mine = {}
        for r, named in tensors.items():
            mine[r] = {}
            for name, t in named.items():
                entry = {"ptr": t.data_ptr()}
                if self.distributed:
                    h = ctypes.create_string_buffer(64)
                    off = ctypes.c_int64(0)
                    nat.check(nat.lib().tps_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)), "ipc_get_handle")
                    entry.update(handle=bytes(h.raw), offset=off.value)
                mine[r][name] = entry
        out: dict[int, dict[str, int]] = {}
        for table in self.allgather(mine):
            for r, named in table.items():
                out[r] = {}
                for name, e in named.items():
                    if r in self.local_ranks:
                        out[r][name] = e["ptr"]
                    else:
                        key = e["handle"]
                        if key not in self._ipc_cache:
                            base = ctypes.c_void_p(0)
                            nat.check(nat.lib().tps_ipc_open(key, ctypes.byref(base)), "ipc_open")
                            self._ipc_cache[key] = base.value
                        out[r][name] = self._ipc_cache[key] + e["offset"]
        return out


    def close_peers(self) -> None:
        """Unmap every peer buffer this process opened (tps_ipc_close) and forget the handles.
        For discarding a whole backend: call it on every rank after the last kernel that touches
        a peer buffer (device synchronised, then a barrier) and before any rank frees memory it
        exported (another barrier) -- freeing an exported buffer that a peer still has mapped is
        undefined in CUDA IPC, and its memory is not reclaimed while the mapping lives."""
        for base in self._ipc_cache.values():
            nat.check(nat.lib().tps_ipc_close(base), "ipc_close")
        self._ipc_cache.clear()


class CacheManager:
    """Per-layout communicator tables, created on first use and kept (grow-only pool)."""

    def __init__(self, world: World, max_batch: int, hidden: int, n_phases: int):
        self.world = world
        self.max_batch = max_batch
        self.hidden = hidden
        self.n_phases = n_phases
        self.pool: dict[int, dict[int, GroupComm]] = {}
        self.created: list[int] = []

    def get(self, tp: int) -> dict[int, GroupComm | None]:
        """{local rank: GroupComm} for TP degree tp (None entries for tp == 1)."""
        if tp == 1:
            return {r: None for r in self.world.local_ranks}
        if tp in self.pool:
            return self.pool[tp]
        comms = {r: GroupComm(tp, r % tp, self.max_batch, self.hidden, self.n_phases, self.world.devices[r])
                 for r in self.world.local_ranks}
        ptrs = self.world.share({r: {"recv": c.recv, "ll": c.ll, "ctr": c.ctr, "cand": c.cand, "am": c.am}
                                 for r, c in comms.items()})
        for r, c in comms.items():
            g0 = (r // tp) * tp
            c.connect([ptrs[g0 + i] for i in range(tp)])
        self.pool[tp] = comms
        self.created.append(tp)
        return comms
