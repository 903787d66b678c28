"""Assembly of one DP group's ranks: shards, KV pools, slot tables, executors.

`build_group` creates the `tp` ranks of one group on a single device (tp == 1:
the normal one-GPU worker; tp > 1: a *virtual* TP group whose ranks share the
GPU and whose "peer" pointers are plain device pointers -- the same kernels and
counter protocol as the NVLink path, used by the single-GPU tests and the
Switch Executor microbench). The multi-process path builds one rank per
process and connects the GroupComm tables through CUDA IPC (cache_manager).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as nat
from .executor import GroupComm, GroupRunner, InferExecutor
from .kvcache import KVPool, SlotTable, pages_for
from .models import DecoderGeometry, rank_shard
from .shards import RankWeights
from .workload import as_int64


@dataclass
class RankState:
    weights: RankWeights
    kv: KVPool
    slots: SlotTable
    executor: InferExecutor
    comm: GroupComm | None


def n_phases(geom: DecoderGeometry) -> int:
    return 2 * geom.num_layers + 1


def build_rank(geom: DecoderGeometry, tp: int, rank: int, max_batch: int, num_slots: int, max_len: int,
               device, seed: int | None = 0, kv_pages: int | None = None,
               weights: RankWeights | None = None, prefill_rows: int = 0) -> RankState:
    nat.init_device(torch.device(device).index or 0)
    sh = rank_shard(geom, tp, rank)
    if weights is None:
        weights = RankWeights(geom, sh, device)
        if seed is not None:
            weights.fill_random(seed)
    if kv_pages is None:
        kv_pages = num_slots * pages_for(max_len)
    kv = KVPool(geom.num_layers, sh.n_kv, geom.head_dim, kv_pages, device)
    slots = SlotTable(num_slots, max_len, device)
    comm = None
    if tp > 1:
        comm = GroupComm(tp, rank, max(max_batch, prefill_rows), geom.hidden, n_phases(geom), torch.device(device))
    ex = InferExecutor(geom, sh, weights, kv, slots, max_batch, device, comm=comm, prefill_rows=prefill_rows)
    return RankState(weights, kv, slots, ex, comm)


def connect_virtual(ranks: list[RankState]) -> None:
    if len(ranks) == 1:
        return
    tables = [r.comm.export() for r in ranks]
    for r in ranks:
        r.comm.connect(tables)


def build_group(geom: DecoderGeometry, tp: int, max_batch: int, num_slots: int, max_len: int,
                device="cuda:0", seed: int | None = 0, use_graphs: bool = True):
    ranks = [build_rank(geom, tp, r, max_batch, num_slots, max_len, device, seed) for r in range(tp)]
    connect_virtual(ranks)
    runner = GroupRunner([r.executor for r in ranks], use_graphs=use_graphs)
    return ranks, runner


def admit(ranks: list[RankState], sample_id: int, prompt: list[int], max_ctx: int,
          slot: int | None = None, seed: int = 0) -> int:
    """Place a sample on every rank of its group: slot, reserved pages, prompt tokens.

    Pages are reserved for max_ctx tokens (prompt + l_max), the reference's
    admission rule (tpshift/engine.py:142-147). Ranks allocate in lock-step, so
    the slot index is the same on every rank of the group.
    """
    n_pages = pages_for(max_ctx)
    got = None
    if not isinstance(prompt, torch.Tensor):
        prompt = torch.tensor(prompt, dtype=torch.int32)
    for r in ranks:
        s = r.slots.alloc(sample_id) if slot is None else slot
        if got is not None and s != got:
            raise RuntimeError("slot tables of a TP group diverged")
        got = s
        if n_pages > r.slots.max_pages:
            raise ValueError("max_ctx exceeds the slot table's max_len")
        pages = r.kv.alloc(n_pages)
        r.slots.pages[s] = pages
        h2d(r.slots.page_table[s, :n_pages], pages)
        r.slots.history[s, :prompt.numel()].copy_(prompt, non_blocking=True)
        r.slots.pos[s] = 0
        r.slots.seed[s] = as_int64(seed)
        r.executor.prompt_len[s] = prompt.numel()
    return got


def h2d(dst: torch.Tensor, values) -> None:
    """Asynchronous small host->device write through pinned memory (never syncs the stream)."""
    host = torch.as_tensor(values, dtype=dst.dtype)
    if dst.device.type == "cuda":
        host = host.pin_memory()
    dst.copy_(host, non_blocking=True)


def retire(ranks: list[RankState], slot: int) -> None:
    for r in ranks:
        r.kv.release(r.slots.pages.get(slot, []))
        r.slots.release(slot)


def last_logits(ranks: list[RankState]) -> torch.Tensor:
    """fp32 logits [B, V] of the last eagerly issued step (vocab shards in rank order)."""
    outs = []
    for r in ranks:
        ex = r.executor
        srcs, B = ex._last_lm_srcs
        out = torch.empty((B, ex.V), dtype=torch.float32, device=ex.device)
        nat.check(nat.lib().tps_sum_partials(*srcs, B * ex.V, out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream), "tps_sum_partials")
        outs.append(out)
    return torch.cat(outs, dim=1)
