"""Infer Executor: one TP rank's decode step on the sm_100a engine.

Replaces the reference's per-round latency oracle (the n-round block at
tpshift/engine.py:287-300 prices `oracle_decode_latency(hw, tp, B, T)`,
tpshift/latency.py:111-133) with the real step:

  embed -> [ RMSNorm -> QKV (tcgen05) -> bias+RoPE+KV-append -> paged attention
             -> O (tcgen05) -> TP allreduce -> add+RMSNorm -> gate/up (tcgen05)
             -> SiLU*up -> down (tcgen05) -> TP allreduce -> add+RMSNorm ] x L
        -> LM head (tcgen05, vocab-parallel) -> argmax (+ cross-rank reduce)

A step is written once as a *program* (a Python generator that issues the
rank's launches and yields at every point where it would wait for TP peers).
One process per GPU runs its own program straight through (peers are NVLink
mappings and device counters do the waiting); a single-GPU "virtual group"
advances the programs of all ranks in lock-step, so the same kernels and the
same counter protocol run on one device. Each (bucket) program is captured
once into a CUDA graph and replayed for every round of a block.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .kvcache import PAGE, KVPool, SlotTable
from .models import DecoderGeometry, RankShard, rank_shard, rope_tables
from .shards import RankWeights

BUCKETS = (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256)


def bucket_for(b: int, max_batch: int) -> int:
    for x in BUCKETS:
        if x >= b:
            return min(x, max_batch) if x > max_batch else x
    return max_batch


PREFILL_GROUP_MAX = 16  # positions per group of the grouped prefill attention (tps_prefill_attention)


def prefill_groups(row_slot, gp: int) -> tuple[np.ndarray, np.ndarray]:
    """Group table of a prefill chunk: the rows of each sample (row_slot >= 0) in chunk order,
    cut into groups of at most `gp` positions -> (rows int32 [R][16] (-1 pad), n int32 [R])."""
    rs = np.asarray(row_slot, dtype=np.int64)
    R = len(rs)
    rows = np.full((R, PREFILL_GROUP_MAX), -1, dtype=np.int32)
    n = np.zeros(R, dtype=np.int32)
    open_grp: dict[int, int] = {}
    ng = 0
    for i, s in enumerate(rs.tolist()):
        if s < 0:
            continue
        gi = open_grp.get(s)
        if gi is None or n[gi] >= gp:
            gi = ng
            ng += 1
            open_grp[s] = gi
        rows[gi, n[gi]] = i
        n[gi] += 1
    return rows, n


def argmax_chunks(B: int) -> int:
    return max(1, min(64, 296 // max(1, B)))


FUSE_ROWS = 64     # tail batches (B <= FUSE_ROWS) exchange the TP allreduce as LL {value, tag} pairs
LL_EPILOGUE_ROWS = 16  # ... from the projection epilogue (every split partial) up to this batch; above it
                       # a reduce kernel sums the splits first (S x fewer NVLink bytes; the crossover of
                       # the extra launch vs the modeled NVLink bytes is ~16 rows at TP8)
# B <= LL_CLUSTER_ROWS: the projection's split-K CTAs reduce over DSMEM inside the kernel and
# push one LL pair per element (tps_linear_push_ll_cluster; supersedes both forms above)
LL_CLUSTER_ROWS = int(os.environ.get("TPS_LL_CLUSTER_ROWS", "64"))
# ... at TP >= 4 (TP2 shards are large enough that the one-wave cluster split -- 4-stage ring,
# S <= 148 / tiles -- streams slower than the 8-stage per-partial form: Qwen2.5-32B fixed TP2
# stage 63.4 -> 65.5 s predicted; Qwen2.5-7B TP2 B <= 32 +2-3 % in loopback)
LL_CLUSTER_MIN_TP = 4
FUSE_SOURCES = 16  # LL slots per parity: tp x splits partials of one fused allreduce (one load batch)
# persistent decode step (csrc/persist.cu): one launch per step for B <= PERSIST_MAX_ROWS.
# Parity-green but measured slower than the per-kernel step on B200 (TP8 B=1 1.80 vs 1.30 ms,
# TP1 B=1 4.28 vs 3.00 ms): opt-in (TPS_PERSIST=1 or use_persist)
PERSIST_MAX_ROWS = 16
PERSIST = os.environ.get("TPS_PERSIST", "0") == "1"
# B <= GEMV_ROWS: every projection of the step on the CUDA-core warp-shuffle GEMV
# (csrc/gemv.cu; same output contracts as the tcgen05 forms, at most tps_gemv_max_rows() = 4
# rows). Opt-in (TPS_GEMV_ROWS=4 or InferExecutor.gemv_rows) until it is measured against the
# tcgen05 tail on B200: bench.py's `tail` section times both.
GEMV_ROWS = int(os.environ.get("TPS_GEMV_ROWS", "0"))


class GroupComm:
    """Communication state of one TP group as held by one rank.

    recv[parity][src_rank] : fp32 [max_batch][H] receive slots (one-shot allreduce push)
    ll[parity][src_rank * splits + split] : uint64 [FUSE_ROWS][H] {fp32, tag} slots the peers'
                             fused projection epilogues store their split partials into (LL)
    cand                   : per-(row, chunk) argmax candidates (8 B each)
    ctr[phase]             : arrival counters, +1 per peer per phase per step
    done[phase]            : last-CTA detectors of this rank's signalling launches
    epoch                  : step counter; waits target epoch * tp
    """

    def __init__(self, tp: int, rank: int, max_batch: int, hidden: int, n_phases: int,
                 device: torch.device):
        self.tp = tp
        self.rank = rank
        self.max_batch = max_batch
        self.hidden = hidden
        self.n_phases = n_phases
        self.recv = torch.zeros((2, tp, max_batch, hidden), dtype=torch.float32, device=device)
        # tags start at 0 and live tags are >= n_phases (epochs start at 1): no stale match
        self.ll = torch.zeros((2, FUSE_SOURCES, FUSE_ROWS, hidden), dtype=torch.int64, device=device)
        self.cand = torch.zeros((max_batch, 64, 2), dtype=torch.int32, device=device)
        # persistent step's argmax exchange: LL {value, tag} / {index, tag} per (parity, src, row)
        self.am = torch.zeros((2, 8, PERSIST_MAX_ROWS, 2), dtype=torch.int64, device=device)
        self.ctr = torch.zeros(n_phases, dtype=torch.int64, device=device)
        self.done = torch.zeros(n_phases, dtype=torch.int32, device=device)
        self.epoch = torch.ones(1, dtype=torch.int64, device=device)
        # peer pointer table, rank order (filled by connect / the Cache Manager)
        self.peer_recv: list[int] = []
        self.peer_ll: list[int] = []
        self.loopback = False  # timing harness: this rank plays every peer of its group
        self.peer_ctr: list[int] = []
        self.peer_cand: list[int] = []
        self.peer_am: list[int] = []

    # local export for peers
    def export(self) -> dict:
        return {"recv": self.recv.data_ptr(), "ll": self.ll.data_ptr(), "ctr": self.ctr.data_ptr(),
                "cand": self.cand.data_ptr(), "am": self.am.data_ptr()}

    def connect(self, tables: list[dict]) -> None:
        assert len(tables) == self.tp
        self.peer_recv = [t["recv"] for t in tables]
        self.peer_ll = [t["ll"] for t in tables]
        self.peer_ctr = [t["ctr"] for t in tables]
        self.peer_cand = [t["cand"] for t in tables]
        self.peer_am = [t["am"] for t in tables]

    def recv_slot(self, base: int, parity: int, src_rank: int) -> int:
        return base + ((parity * self.tp + src_rank) * self.max_batch * self.hidden) * 4

    def ll_slot(self, base: int, parity: int, src_rank: int, splits: int) -> int:
        """First slot of src_rank in an LL receive area when every rank pushes `splits`
        partials: slot index src_rank * splits + split, so the tp x splits used slots are
        contiguous and are read back in (rank, split) order."""
        return base + ((parity * FUSE_SOURCES + src_rank * splits) * FUSE_ROWS * self.hidden) * 8

    def reset(self) -> None:
        # the epoch restarts at 1: clear the LL slots too, or a tag stored before the reset
        # (epoch e, phase p) would satisfy the same (e, p) wait after it
        self.ctr.zero_()
        self.done.zero_()
        self.ll.zero_()
        self.am.zero_()
        self.epoch.fill_(1)


@dataclass
class LaunchStats:
    kernels: int = 0
    by_kind: dict = field(default_factory=dict)

    def add(self, kind: str, n: int = 1) -> None:
        self.kernels += n
        self.by_kind[kind] = self.by_kind.get(kind, 0) + n


class InferExecutor:
    """Decode-step engine of one TP rank (the per-GPU Infer Executor)."""

    def __init__(self, geom: DecoderGeometry, shard: RankShard, weights: RankWeights, kv: KVPool,
                 slots: SlotTable, max_batch: int, device: torch.device | str,
                 comm: GroupComm | None = None, stream: torch.cuda.Stream | None = None,
                 prefill_rows: int = 0):
        self.geom = geom
        self.shard = shard
        self.w = weights
        self.kv = kv
        self.slots = slots
        self.max_batch = max_batch
        # chunked prefill runs `prefill_rows` (sample, prompt position) rows per step
        self.prefill_rows = prefill_rows
        rows = max(max_batch, prefill_rows)
        # launch kinds left out of the step program (timing probes only: results are garbage)
        self.skip: frozenset = frozenset()
        # 0: greedy; > 0: Gumbel-max sampling at this temperature with the slots' Philox keys
        self.temperature = 0.0
        # gate/up with the SwiGLU fused (split-K 1) once this many (tile x act) units exist
        self.fuse_silu_min_units = 120
        self.device = torch.device(device)
        self.comm = comm
        self.tp = shard.tp
        self.rank = shard.rank
        assert (self.tp == 1) == (comm is None), "TP>1 needs a GroupComm"
        nat.lib()
        H, D = geom.hidden, geom.head_dim
        self.nq, self.nkv = shard.n_q, shard.n_kv
        self.n_qkv = (self.nq + 2 * self.nkv) * D
        self.F = shard.ffn_width
        self.V = shard.vocab_width
        dev = self.device
        cos, sin = rope_tables(geom, slots.max_len + 1)
        self.cos = torch.from_numpy(cos).to(dev)
        self.sin = torch.from_numpy(sin).to(dev)
        self.resid = torch.zeros((rows, H), dtype=torch.float32, device=dev)
        self.xn = torch.zeros((rows, H), dtype=torch.bfloat16, device=dev)
        self.q = torch.zeros((rows, self.nq, D), dtype=torch.bfloat16, device=dev)
        self.attn = torch.zeros((rows, self.nq * D), dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros((rows, self.F), dtype=torch.bfloat16, device=dev)
        self.prompt_len = torch.zeros(slots.num_slots, dtype=torch.int32, device=dev)
        sizes = self.buckets() + ([prefill_rows] if prefill_rows else [])
        # split-K workspace sized for the worst projection over all row counts
        ws = 0
        for B in sizes:
            for n, k in self._proj_shapes():
                ws = max(ws, nat.lib().tps_linear_splits(n, k, B) * B * n)
        self.ws = torch.zeros(ws, dtype=torch.float32, device=dev)
        # attention partial states: the page-balanced schedule (nsplit 0) and a fixed split
        # count for every bucket (the policy's own count, else one wave of 2 CTAs per SM)
        att = max(nat.lib().tps_attn_workspace(B, self.nq, D, s) for B in sizes
                  for s in (0, self._fixed_attn_splits(B)))
        self.att_o = torch.zeros(att, dtype=torch.float32, device=dev)
        self.att_m = torch.zeros(att // D, dtype=torch.float32, device=dev)
        self.att_l = torch.zeros_like(self.att_m)
        self.att_ctr = torch.zeros(rows * self.nkv, dtype=torch.int32, device=dev)
        self.local_cand = torch.zeros((max_batch, 64, 2), dtype=torch.int32, device=dev)
        # TP1 greedy: the LM head's epilogue emits one candidate per (row, 128-column tile)
        self.lm_argmax = os.environ.get("TPS_LM_ARGMAX", "1") == "1"
        self.lm_tiles = -(-self.w[(-1, "lm_head")].shape[0] // 128)
        self.lm_cand = torch.zeros((max_batch, self.lm_tiles, 2), dtype=torch.int32, device=dev)
        self.out_tok = torch.zeros(max_batch, dtype=torch.int32, device=dev)
        self.row_slot = {B: torch.full((B,), -1, dtype=torch.int32, device=dev) for B in sizes}
        self.row_pos = {prefill_rows: torch.zeros(prefill_rows, dtype=torch.int32, device=dev)} \
            if prefill_rows else {}
        # grouped prefill attention: one CTA per (sample group, KV head) reads the sample's
        # pages once for all its rows in the chunk (else every row is its own segment)
        self.group_positions = nat.lib().tps_prefill_group_positions(self.nq // self.nkv) \
            if self.nq % self.nkv == 0 else 0
        self.prefill_grouped = self.group_positions > 0
        if prefill_rows:
            self.grp_rows = torch.full((prefill_rows, PREFILL_GROUP_MAX), -1, dtype=torch.int32, device=dev)
            self.grp_n = torch.zeros(prefill_rows, dtype=torch.int32, device=dev)
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self.launch_stats: dict[int, LaunchStats] = {}
        # persistent step (csrc/persist.cu) state: workspace, logits, CTAs per rank it was sized for
        self.use_persist = PERSIST
        self.gemv_rows = min(GEMV_ROWS, nat.lib().tps_gemv_max_rows())
        self.p_work: torch.Tensor | None = None
        self.p_logits: torch.Tensor | None = None
        self.p_ctas = 0
        self.p_trace: torch.Tensor | None = None   # tools/persist_trace.py
        self.p_trace_layer = -1

    # ------------------------------------------------------------ shapes ---
    def buckets(self) -> list[int]:
        out = [b for b in BUCKETS if b <= self.max_batch]
        if not out or out[-1] != self.max_batch:
            out.append(self.max_batch)
        return out

    def bucket(self, b: int) -> int:
        for x in self.buckets():
            if x >= b:
                return x
        raise ValueError(f"batch {b} exceeds max_batch {self.max_batch}")

    def _proj_shapes(self):
        g = self.geom
        return [(self.n_qkv, g.hidden), (g.hidden, self.nq * g.head_dim), (2 * self.F, g.hidden),
                (g.hidden, self.F), (self.V, g.hidden)]

    # --------------------------------------------------------- primitives ---
    def _splits(self, n: int, k: int, B: int) -> int:
        return nat.lib().tps_linear_splits(n, k, B)

    def _fuse_silu(self, B: int) -> bool:
        """SwiGLU in the gate/up epilogue needs split-K = 1: worth it when the 128-row
        tiles (x activation tiles) alone fill most of the 148 SMs."""
        bn = 16 if B <= 16 else 32 if B <= 32 else 64 if B <= 64 else 128 if B <= 128 else 256
        units = (2 * self.F // 128) * (-(-B // bn))
        return units >= self.fuse_silu_min_units

    def _fixed_attn_splits(self, B: int) -> int:
        s = self._attn_splits(B)
        return s if s > 0 else max(1, min(32, 2 * 148 // (B * self.nkv)))

    def _attn_splits(self, B: int) -> int:
        """tps_attn_splits policy (-1 = cluster per segment, 0 = page-balanced, n = fixed splits)."""
        return nat.lib().tps_attn_splits(B, self.nkv, self.slots.max_pages)

    def _linear(self, st, stats, w: torch.Tensor, x: torch.Tensor, B: int) -> tuple[int, int, int]:
        """Projection into the split-K workspace; returns the strided source (base, n, stride)."""
        n, k = w.shape
        s = self._splits(n, k, B)
        if "linear" in self.skip:
            return (self.ws.data_ptr(), s, B * n)
        if B <= self.gemv_rows:
            nat.check(nat.lib().tps_gemv(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[1], self.ws.data_ptr(), st),
                      "tps_gemv")
            stats.add("linear")
            return (self.ws.data_ptr(), 1, B * n)
        nat.check(nat.lib().tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0],
                                       x.shape[1], self.ws.data_ptr(), s, st), "tps_linear")
        stats.add("linear")
        return (self.ws.data_ptr(), s, B * n)

    @staticmethod
    def _arr(ptrs):
        # host pointer list, consumed (copied into a by-value kernel parameter) by the call
        return nat.ptr_array(ptrs)

    def set_prefill_rows(self, rs: torch.Tensor, rp: torch.Tensor, gp: int = 0) -> None:
        """Bind a prefill chunk (CPU int32 [prefill_rows] row slots / positions, pinned for an
        asynchronous copy) and its sample-group table (`gp` positions per group, default this
        executor's maximum)."""
        R = self.prefill_rows
        self.row_slot[R].copy_(rs, non_blocking=True)
        self.row_pos[R].copy_(rp, non_blocking=True)
        if self.prefill_grouped:
            rows, n = prefill_groups(rs.numpy(), gp or self.group_positions)
            self.grp_rows.copy_(torch.from_numpy(rows).pin_memory(), non_blocking=True)
            self.grp_n.copy_(torch.from_numpy(n).pin_memory(), non_blocking=True)

    # ------------------------------------------------------------ program ---
    def program(self, B: int, st: int, stats: LaunchStats | None = None, prefill: bool = False):
        """Issue one decode step for bucket B on stream `st`; yields at peer waits.

        prefill=True: B = prefill_rows (sample, prompt position) rows bound by
        set_prefill_rows; the layers run exactly as in decode (K/V of every row
        appended before attention, each row attending causally to positions <=
        its own), and the LM head / argmax are skipped.
        """
        stats = stats if stats is not None else LaunchStats()
        lib = nat.lib()
        g = self.geom
        H, D, L = g.hidden, g.head_dim, g.num_layers
        W = self.w
        sl = self.slots
        rs = self.row_slot[B].data_ptr()
        rp = self.row_pos[B].data_ptr() if prefill else None
        pos = sl.pos.data_ptr()
        hist = sl.history.data_ptr()
        eps = ctypes.c_float(g.rms_eps)

        nat.check(lib.tps_embed(rs, pos, rp, hist, sl.max_len, W.tensor_ptr(-1, "embed"), H, B,
                                self.resid.data_ptr(), st), "tps_embed")
        stats.add("embed")
        nat.check(lib.tps_add_norm(self.resid.data_ptr(), None, 0, 0, None, W.tensor_ptr(0, "ln1"), eps,
                                   H, B, self.xn.data_ptr(), H, st), "tps_add_norm")
        stats.add("add_norm")
        nsplit = self._attn_splits(B)
        for l in range(L):
            kc, vc = self.kv.layer_ptrs(l)
            bias = W.tensor_ptr(l, "b_qkv") if g.qkv_bias else None
            srcs = self._linear(st, stats, W[(l, "w_qkv")], self.xn, B)
            if "qkv_rope" not in self.skip:
                # bias + RoPE + paged KV append (prefill: every row's K/V appended before attention)
                nat.check(lib.tps_qkv_rope_append(*srcs, bias, rs, pos, rp,
                                                  sl.page_table.data_ptr(), sl.max_pages,
                                                  self.cos.data_ptr(), self.sin.data_ptr(), B, self.nq,
                                                  self.nkv, D, PAGE, self.q.data_ptr(), kc, vc, st),
                          "tps_qkv_rope_append")
                stats.add("qkv_rope_append")
            if "attention" not in self.skip and prefill and self.prefill_grouped:
                nat.check(lib.tps_prefill_attention(self.q.data_ptr(), kc, vc, rs, rp, self.grp_rows.data_ptr(),
                                                    self.grp_n.data_ptr(), B, sl.page_table.data_ptr(), sl.max_pages,
                                                    self.nq, self.nkv, D, self.attn.data_ptr(), st),
                          "tps_prefill_attention")
                stats.add("paged_attention")
            elif "attention" not in self.skip:
                nat.check(lib.tps_paged_attention(self.q.data_ptr(), kc, vc, rs, pos, rp, sl.page_table.data_ptr(),
                                                  sl.max_pages, B, self.nq, self.nkv, D, nsplit,
                                                  self.att_m.data_ptr(), self.att_l.data_ptr(),
                                                  self.att_o.data_ptr(), self.att_ctr.data_ptr(),
                                                  self.attn.data_ptr(), None, 0, 0, None, None, None, st),
                          "tps_paged_attention")
                stats.add("paged_attention", 1 if nsplit <= 4 else 2)  # (+ split-merge kernel)
            yield from self._row_parallel(st, stats, 2 * l, "w_o", W[(l, "w_o")], self.attn, B,
                                          W.tensor_ptr(l, "ln2"))
            w_gu = W[(l, "w_gu")]
            if B <= self.gemv_rows and "linear" not in self.skip:
                nat.check(lib.tps_gemv_silu(w_gu.data_ptr(), 2 * self.F, H, H, self.xn.data_ptr(), B, H,
                                            self.act.data_ptr(), self.F, st), "tps_gemv_silu")
                stats.add("linear")
            elif self._fuse_silu(B):
                nat.check(lib.tps_linear_silu(w_gu.data_ptr(), 2 * self.F, H, H, self.xn.data_ptr(), B,
                                              self.xn.shape[0], H, self.act.data_ptr(), self.F, st),
                          "tps_linear_silu")
                stats.add("linear")
            else:
                srcs = self._linear(st, stats, w_gu, self.xn, B)
                if "silu" not in self.skip:
                    nat.check(lib.tps_silu_mul(*srcs, B, self.F, self.act.data_ptr(), self.F, st),
                              "tps_silu_mul")
                    stats.add("silu_mul")
            nxt = W.tensor_ptr(l + 1, "ln1") if l + 1 < L else W.tensor_ptr(-1, "ln_f")
            yield from self._row_parallel(st, stats, 2 * l + 1, "w_d", W[(l, "w_d")], self.act, B, nxt)
        cm = self.comm
        if prefill:
            if cm is not None:
                # keep every phase counter in step with the epoch: an empty push that
                # only signals the argmax phase, then advance the epoch
                ph = 2 * L
                sigs = [p + ph * 8 for p in cm.peer_ctr]
                nat.check(lib.tps_reduce_push(self.ws.data_ptr(), 1, 0, self._arr([self.ws.data_ptr()]), 1, 0,
                                              self._arr(sigs), len(sigs), cm.done.data_ptr() + ph * 4, st),
                          "tps_reduce_push")
                nat.check(lib.tps_epoch_advance(cm.epoch.data_ptr(), st), "tps_epoch_advance")
                stats.add("reduce_push")
                stats.add("epoch_advance")
            return
        if cm is None and self.temperature <= 0 and self.lm_argmax and "linear" not in self.skip:
            w = W[(-1, "lm_head")]
            if B <= self.gemv_rows:
                nat.check(lib.tps_gemv_argmax(w.data_ptr(), w.shape[0], w.shape[1], w.shape[1], self.xn.data_ptr(), B,
                                              self.xn.shape[1], self.ws.data_ptr(), self.lm_cand.data_ptr(),
                                              self.shard.vocab[0], st), "tps_gemv_argmax")
            else:
                nat.check(lib.tps_linear_argmax(w.data_ptr(), w.shape[0], w.shape[1], w.shape[1], self.xn.data_ptr(),
                                                B, self.xn.shape[0], self.xn.shape[1], self.ws.data_ptr(),
                                                self.lm_cand.data_ptr(), self.shard.vocab[0], st), "tps_linear_argmax")
            stats.add("linear")
            self._last_lm_srcs = ((self.ws.data_ptr(), 1, B * w.shape[0]), B)
            nat.check(lib.tps_argmax_finalize(self._arr([self.lm_cand.data_ptr()]), 1, self.lm_tiles, None, B, rs,
                                              pos, self.prompt_len.data_ptr(), hist, sl.max_len,
                                              self.out_tok.data_ptr(), st), "tps_argmax_finalize")
            stats.add("argmax_finalize")
            return
        srcs = self._linear(st, stats, W[(-1, "lm_head")], self.xn, B)
        self._last_lm_srcs = (srcs, B)
        nch = argmax_chunks(B)
        if cm is None:
            self._stage1(srcs, B, nch, self.local_cand.data_ptr(), None, 0, None, rs, pos, st)
            stats.add("argmax_stage1")
            cands = [self.local_cand.data_ptr()]
            wait = None
        else:
            ph = 2 * L
            sigs = [p + ph * 8 for p in cm.peer_ctr]
            self._stage1(srcs, B, nch, cm.cand.data_ptr(), self._arr(sigs), len(sigs), cm.done.data_ptr() + ph * 4,
                         rs, pos, st)
            stats.add("argmax_stage1")
            yield
            cands = list(cm.peer_cand)
            wait = nat.wait_spec(cm.ctr.data_ptr() + ph * 8, cm.epoch.data_ptr(), cm.tp, 0)
        nat.check(lib.tps_argmax_finalize(self._arr(cands), len(cands), nch, wait, B, rs, pos,
                                          self.prompt_len.data_ptr(), hist, sl.max_len,
                                          self.out_tok.data_ptr(), st), "tps_argmax_finalize")
        stats.add("argmax_finalize")
        if cm is not None:
            nat.check(lib.tps_epoch_advance(cm.epoch.data_ptr(), st), "tps_epoch_advance")
            stats.add("epoch_advance")

    def _stage1(self, srcs, B, nch, cand, sigs, nsig, done, rs, pos, st):
        """Per-rank candidates over the vocab slice: greedy argmax, or Gumbel-max sampling."""
        lib = nat.lib()
        if self.temperature > 0:
            nat.check(lib.tps_sample_stage1(*srcs, B, self.V, self.shard.vocab[0], nch, cand, sigs, nsig, done,
                                            self.slots.seed.data_ptr(), rs, pos, None,
                                            ctypes.c_float(self.temperature), st), "tps_sample_stage1")
        else:
            nat.check(lib.tps_argmax_stage1(*srcs, B, self.V, self.shard.vocab[0], nch, cand, sigs, nsig, done, st),
                      "tps_argmax_stage1")

    def fused_splits(self, fam: str, B: int) -> int:
        """Split-K count of a fused row-parallel projection: the same on every rank of the
        group (the slots are read as tp x splits partials in one fixed order), with at most
        FUSE_SOURCES partial slots in total (one consumer load batch)."""
        g = self.geom
        if fam == "w_o":
            ks = [rank_shard(g, self.tp, r).n_q * g.head_dim for r in range(self.tp)]
        else:
            ks = [self.F] * self.tp
        s = nat.lib().tps_linear_splits(g.hidden, max(ks), B)
        # (measured: 32 slots for the long-K down projection -- more CTAs, but a second load
        # batch in the consumer -- was slower at TP8 B=1..16)
        return max(1, min(FUSE_SOURCES // self.tp, s, min(-(-k // 64) for k in ks)))

    def _row_parallel(self, st, stats, phase: int, fam: str, w: torch.Tensor, x: torch.Tensor, B: int,
                      norm_w: int):
        """O / down projection + TP allreduce + residual add + RMSNorm.

        TP > 1 and B <= FUSE_ROWS: the projection epilogue stores its split-K partials
        straight into every peer's receive area as {value, tag} pairs (tps_linear_push_ll:
        the allreduce is fused into the projection, LL protocol -- no counters or fences);
        add+norm polls the tags and sums the tp x splits slots in (rank, split) order.
        Otherwise: split partials -> tps_reduce_push -> add+norm."""
        cm = self.comm
        if cm is None or B > FUSE_ROWS or "fuse_push" in self.skip or "linear" in self.skip:
            srcs = self._linear(st, stats, w, x, B)
            yield from self._allreduce_norm(st, stats, phase, srcs, B, norm_w)
            return
        lib = nat.lib()
        g = self.geom
        H = g.hidden
        n, k = w.shape
        par = phase % 2
        # LL: {value, tag} stores polled by the consumer; tag = epoch * n_phases + phase
        # (a loopback timing rank -- profiler.loopback_rank -- fills every rank's slots itself)
        if B <= self.gemv_rows:
            S = 1  # one full dot product per element, pushed once to every rank
            dsts = [cm.ll_slot(base, par, q if cm.loopback else self.rank, 1) for q, base in enumerate(cm.peer_ll)]
            nat.check(lib.tps_gemv_push_ll(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[1], self._arr(dsts),
                                           len(dsts), cm.epoch.data_ptr(), cm.n_phases, phase, st),
                      "tps_gemv_push_ll")
            stats.add("linear")
        elif B <= LL_CLUSTER_ROWS and cm.tp >= LL_CLUSTER_MIN_TP and lib.tps_cluster_splits(n, k, B) > 0:
            S = 1  # one reduced slot per rank
            dsts = [cm.ll_slot(base, par, q if cm.loopback else self.rank, 1) for q, base in enumerate(cm.peer_ll)]
            nat.check(lib.tps_linear_push_ll_cluster(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                                     self._arr(dsts), len(dsts), cm.epoch.data_ptr(), cm.n_phases,
                                                     phase, st), "tps_linear_push_ll_cluster")
            stats.add("linear")
        elif B <= LL_EPILOGUE_ROWS:
            S = self.fused_splits(fam, B)
            dsts = [cm.ll_slot(base, par, q if cm.loopback else self.rank, S) for q, base in enumerate(cm.peer_ll)]
            nat.check(lib.tps_linear_push_ll(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                             self._arr(dsts), len(dsts), FUSE_ROWS * H, S, cm.epoch.data_ptr(),
                                             cm.n_phases, phase, st), "tps_linear_push_ll")
            stats.add("linear")
        else:
            S = 1  # one summed slot per rank
            srcs = self._linear(st, stats, w, x, B)
            dsts = [cm.ll_slot(base, par, q if cm.loopback else self.rank, 1) for q, base in enumerate(cm.peer_ll)]
            nat.check(lib.tps_reduce_push_ll(*srcs, self._arr(dsts), len(dsts), B * H, cm.epoch.data_ptr(),
                                             cm.n_phases, phase, st), "tps_reduce_push_ll")
            stats.add("reduce_push")
        yield
        if "add_norm" in self.skip:
            return
        nat.check(lib.tps_add_norm_ll(self.resid.data_ptr(), cm.ll_slot(cm.ll.data_ptr(), par, 0, S), cm.tp * S,
                                      FUSE_ROWS * H, cm.epoch.data_ptr(), cm.n_phases, phase, norm_w,
                                      ctypes.c_float(g.rms_eps), H, B, self.xn.data_ptr(), H,
                                      cm.ctr.data_ptr() + phase * 8, cm.tp, st), "tps_add_norm_ll")
        stats.add("add_norm")

    def _allreduce_norm(self, st, stats, phase: int, srcs: tuple[int, int, int], B: int, norm_w: int):
        lib = nat.lib()
        g = self.geom
        H = g.hidden
        eps = ctypes.c_float(g.rms_eps)
        cm = self.comm
        if cm is None:
            if "add_norm" not in self.skip:
                nat.check(lib.tps_add_norm(self.resid.data_ptr(), *srcs, None, norm_w, eps, H,
                                           B, self.xn.data_ptr(), H, st), "tps_add_norm")
                stats.add("add_norm")
            return
        par = phase % 2
        dsts = [cm.recv_slot(base, par, self.rank) for base in cm.peer_recv]
        sigs = [p + phase * 8 for p in cm.peer_ctr]
        nat.check(lib.tps_reduce_push(*srcs, self._arr(dsts), len(dsts), B * H,
                                      self._arr(sigs), len(sigs), cm.done.data_ptr() + phase * 4, st),
                  "tps_reduce_push")
        stats.add("reduce_push")
        yield
        mine = (cm.recv_slot(cm.recv.data_ptr(), par, 0), cm.tp, cm.max_batch * H)
        wait = nat.wait_spec(cm.ctr.data_ptr() + phase * 8, cm.epoch.data_ptr(), cm.tp, 0)
        nat.check(lib.tps_add_norm(self.resid.data_ptr(), *mine, wait, norm_w, eps, H, B,
                                   self.xn.data_ptr(), H, st), "tps_add_norm")
        stats.add("add_norm")

    # ------------------------------------------------ persistent decode step ---
    def persist_geom(self) -> "nat.PersistGeom":
        g = self.geom
        return nat.PersistGeom(num_layers=g.num_layers, hidden=g.hidden, head_dim=g.head_dim,
                               n_phases=2 * g.num_layers + 1, rms_eps=g.rms_eps)

    def persist_ok(self, B: int) -> bool:
        """The step for bucket B can run as one persistent launch (csrc/persist.cu): tail
        batches, head_dim 128, greedy, no timing-probe skips."""
        if not (self.use_persist and B <= PERSIST_MAX_ROWS and self.geom.head_dim == 128
                and self.temperature <= 0 and not self.skip and B in self.row_slot):
            return False
        if self.comm is not None and self.comm.tp > 8:
            return False
        return bool(nat.lib().tps_persist_supported(ctypes.byref(self.persist_geom()),
                                                     ctypes.byref(self._persist_desc(B, 0)[0]), B))

    def _persist_desc(self, B: int, ctas: int):
        """tps_persist_rank of this rank for bucket B (and the host arrays it points to)."""
        g, W, sl = self.geom, self.w, self.slots
        L = g.num_layers
        keep = []

        def arr(ptrs):
            a = nat.ptr_array(ptrs)
            keep.append(a)
            return ctypes.cast(a, ctypes.c_void_p)

        r = nat.PersistRank()
        r.w_qkv = arr([W.tensor_ptr(l, "w_qkv") for l in range(L)])
        r.b_qkv = arr([W.tensor_ptr(l, "b_qkv") for l in range(L)]) if g.qkv_bias else None
        r.w_o = arr([W.tensor_ptr(l, "w_o") for l in range(L)])
        r.w_gu = arr([W.tensor_ptr(l, "w_gu") for l in range(L)])
        r.w_d = arr([W.tensor_ptr(l, "w_d") for l in range(L)])
        r.ln1 = arr([W.tensor_ptr(l, "ln1") for l in range(L)])
        r.ln2 = arr([W.tensor_ptr(l, "ln2") for l in range(L)])
        r.embed = W.tensor_ptr(-1, "embed")
        r.ln_f = W.tensor_ptr(-1, "ln_f")
        r.lm_head = W.tensor_ptr(-1, "lm_head")
        r.k_cache = arr([self.kv.layer_ptrs(l)[0] for l in range(L)])
        r.v_cache = arr([self.kv.layer_ptrs(l)[1] for l in range(L)])
        r.nq, r.nkv, r.ffn, r.vocab, r.vocab_off = self.nq, self.nkv, self.F, self.V, self.shard.vocab[0]
        for q in range(self.tp):
            r.nq_of[q] = rank_shard(g, self.tp, q).n_q
        r.row_slot = self.row_slot[B].data_ptr()
        r.pos = sl.pos.data_ptr()
        r.page_table = sl.page_table.data_ptr()
        r.max_pages = sl.max_pages
        r.history = sl.history.data_ptr()
        r.hist_ld = sl.max_len
        r.prompt_len = self.prompt_len.data_ptr()
        r.out_tok = self.out_tok.data_ptr()
        r.logits = self.p_logits.data_ptr() if self.p_logits is not None else None
        r.cos_t = self.cos.data_ptr()
        r.sin_t = self.sin.data_ptr()
        r.work = self.p_work.data_ptr() if self.p_work is not None else None
        r.work_bytes = self.p_work.numel() if self.p_work is not None else 0
        cm = self.comm
        r.tp = self.tp
        r.rank = self.rank
        if cm is not None:
            H = g.hidden
            r.loopback = 1 if cm.loopback else 0
            r.ll_par_stride = FUSE_SOURCES * FUSE_ROWS * H
            r.ll_src_stride = FUSE_ROWS * H
            for q in range(cm.tp):
                r.ll_peer[q] = cm.peer_ll[q]
                r.am_peer[q] = cm.peer_am[q]
            r.ll_mine = cm.ll.data_ptr()
            r.am_mine = cm.am.data_ptr()
            r.epoch = cm.epoch.data_ptr()
            r.ctr = cm.ctr.data_ptr()
        if self.p_trace is not None:  # probe: per-CTA phase marks of one layer
            r.trace = self.p_trace.data_ptr()
            r.trace_layer = self.p_trace_layer
        return r, keep

    def persist_alloc(self, ctas: int) -> None:
        """Workspace (zeroed: step counters start at 0) and logits buffer of the persistent step."""
        if self.p_ctas == ctas:
            return
        r, _ = self._persist_desc(max(b for b in self.row_slot if b <= PERSIST_MAX_ROWS), ctas)
        n = nat.lib().tps_persist_work_bytes(ctypes.byref(self.persist_geom()), ctypes.byref(r), ctas)
        if n < 0:
            raise RuntimeError("tps_persist_work_bytes failed")
        self.p_work = torch.zeros(int(n), dtype=torch.uint8, device=self.device)
        self.p_logits = torch.zeros((PERSIST_MAX_ROWS, self.V), dtype=torch.float32, device=self.device)
        self.p_ctas = ctas

    # ----------------------------------------------------------- batching ---
    def set_rows(self, B: int, slots: list[int]) -> None:
        """Bind batch rows of bucket B to sample slots (padding rows -> -1)."""
        assert len(slots) <= B
        host = torch.full((B,), -1, dtype=torch.int32)
        host[:len(slots)] = torch.tensor(slots, dtype=torch.int32)
        self.row_slot[B].copy_(host.pin_memory() if self.device.type == "cuda" else host,
                               non_blocking=True)


def run_programs(programs) -> None:
    """Advance per-rank step programs in lock-step (single-GPU virtual group)."""
    live = list(programs)
    while live:
        nxt = []
        for p in live:
            try:
                next(p)
                nxt.append(p)
            except StopIteration:
                pass
        live = nxt


class GroupRunner:
    """Drives the executors of one DP group (1 rank, or all ranks of a virtual TP group)."""

    def __init__(self, executors: list[InferExecutor], use_graphs: bool = True):
        self.ex = executors
        self.use_graphs = use_graphs
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self.stats: dict[int, LaunchStats] = {}
        self.stream = torch.cuda.current_stream(executors[0].device)
        self._pctx: dict[int, tuple] = {}          # bucket -> (device launch context, CTAs per rank)
        self._persist_checked: dict[int, bool] = {}

    def set_rows(self, B: int, slots: list[int]) -> None:
        for e in self.ex:
            e.set_rows(B, slots)

    def _issue(self, B: int, st: int) -> LaunchStats:
        if self.persist_ok(B):
            return self._issue_persist(B, st)
        stats = LaunchStats()
        run_programs([e.program(B, st, stats) for e in self.ex])
        return stats

    # ------------------------------------------------ persistent decode step ---
    def persist_ok(self, B: int) -> bool:
        """One persistent launch per step (csrc/persist.cu) when every rank of this runner
        takes the shape and the runner drives the whole group (virtual) or one rank of it."""
        ex0 = self.ex[0]
        if len(self.ex) not in (1, ex0.tp):
            return False
        if B not in self._persist_checked:
            self._persist_checked[B] = all(e.persist_ok(B) for e in self.ex)
        return self._persist_checked[B]

    def persist_ctas(self) -> int:
        sms = torch.cuda.get_device_properties(self.ex[0].device).multi_processor_count
        return sms // len(self.ex)

    def prepare_persist(self, B: int) -> None:
        """Encode the tensor maps / pointer tables of bucket B (synchronous; outside capture)."""
        if B in self._pctx or not self.persist_ok(B):
            return
        ctas = self.persist_ctas()
        descs, keep = [], []
        for e in self.ex:
            e.persist_alloc(ctas)
            r, k = e._persist_desc(B, ctas)
            descs.append(r)
            keep.append(k)
        arr = (nat.PersistRank * len(descs))(*descs)
        geom = self.ex[0].persist_geom()
        n = nat.lib().tps_persist_ctx_bytes(ctypes.byref(geom), len(descs))
        ctx = torch.empty(int(n), dtype=torch.uint8, device=self.ex[0].device)
        nat.check(nat.lib().tps_persist_prepare(ctypes.byref(geom), arr, len(descs), B, ctas, ctx.data_ptr(),
                                                torch.cuda.current_stream(self.ex[0].device).cuda_stream),
                  "tps_persist_prepare")
        self._pctx[B] = (ctx, ctas)

    def _issue_persist(self, B: int, st: int) -> LaunchStats:
        if B not in self._pctx:
            self.prepare_persist(B)
        ctx, ctas = self._pctx[B]
        nat.check(nat.lib().tps_persist_launch(ctx.data_ptr(), len(self.ex), ctas, B, st), "tps_persist_launch")
        for e in self.ex:
            e._last_lm_srcs = ((e.p_logits.data_ptr(), 1, B * e.V), B)
        stats = LaunchStats()
        stats.add("persist_step")
        return stats

    def capture(self, B: int) -> None:
        """Capture bucket B's step program into a CUDA graph.

        Captured on a private side stream without a device synchronize, so a
        coordinator running ahead of the GPU can capture while earlier rounds
        are still queued. No warm-up run is needed (a step mutates positions):
        kernel attributes are configured once by tps_init.
        """
        if B in self.graphs:
            return
        self.prepare_persist(B)  # (synchronous setup must not run inside the capture)
        g = torch.cuda.CUDAGraph()
        if not hasattr(self, "_cap_stream"):
            self._cap_stream = torch.cuda.Stream(self.ex[0].device)
        s = self._cap_stream
        with torch.cuda.stream(s):
            g.capture_begin()
            try:
                self.stats[B] = self._issue(B, s.cuda_stream)
            finally:
                g.capture_end()
        self.graphs[B] = g

    def step(self, B: int, n: int = 1) -> None:
        """Run n decode rounds for bucket B (rows bound by set_rows)."""
        if self.use_graphs and B in self.graphs:
            g = self.graphs[B]
            for _ in range(n):
                g.replay()
            return
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(n):
            self.stats[B] = self._issue(B, st)

    def kernels_per_step(self, B) -> int:
        return self.stats[B].kernels if B in self.stats else 0

    # ------------------------------------------------------ chunked prefill ---
    def prefill(self, slots: list[int], lengths) -> int:
        """Process positions 0 .. n_i-1 of every slot through the decode kernels
        (n_i = lengths[i], or lengths - 1 for every slot when an int prompt length is
        given: the last prompt position is decode round 1, matching the reference's
        round accounting). Rows are (slot, position) pairs in position-major order,
        `prefill_rows` per step; each step's K/V are appended before its attention, so
        every row attends causally. The tokens must already be in the history table.
        Afterwards every slot's decode position is n_i. Returns kernels launched.

        The ragged form is the recompute path of a switch (tpshift/switchcost.py:203-219):
        a migrated sample's KV is rebuilt from its prompt + generated tokens under the
        target TP instead of being copied."""
        R = self.ex[0].prefill_rows
        if isinstance(lengths, (int, np.integer)):
            lengths = [int(lengths) - 1] * len(slots)
        lengths = [max(0, int(n)) for n in lengths]
        if not slots or max(lengths, default=0) == 0:
            return 0
        if R <= 0:
            raise ValueError("this executor was built without prefill rows")
        rows_s, rows_p = [], []
        for p in range(max(lengths)):
            for s, n in zip(slots, lengths):
                if p < n:
                    rows_s.append(s)
                    rows_p.append(p)
        rows_s = torch.tensor(rows_s, dtype=torch.int32)
        rows_p = torch.tensor(rows_p, dtype=torch.int32)
        key = ("prefill", R)
        kernels = 0
        for k0 in range(0, len(rows_s), R):
            k = min(R, len(rows_s) - k0)
            rs = torch.full((R,), -1, dtype=torch.int32)
            rp = torch.zeros(R, dtype=torch.int32)
            rs[:k] = rows_s[k0:k0 + k]
            rp[:k] = rows_p[k0:k0 + k]
            rs, rp = rs.pin_memory(), rp.pin_memory()
            gp = min(e.group_positions for e in self.ex)
            for e in self.ex:
                e.set_prefill_rows(rs, rp, gp)
            if self.use_graphs:
                if key not in self.graphs:
                    self._capture_key(key, lambda st: self._issue_prefill(R, st))
                self.graphs[key].replay()
            else:
                self.stats[key] = self._issue_prefill(R, torch.cuda.current_stream().cuda_stream)
            kernels += self.kernels_per_step(key)
        idx = torch.tensor(slots, dtype=torch.long).pin_memory()
        val = torch.tensor(lengths, dtype=torch.int32).pin_memory()
        for e in self.ex:  # the next decode round processes position n_i
            e.slots.pos.index_copy_(0, idx.to(e.device, non_blocking=True), val.to(e.device, non_blocking=True))
        return kernels

    def _issue_prefill(self, R: int, st: int) -> LaunchStats:
        stats = LaunchStats()
        run_programs([e.program(R, st, stats, prefill=True) for e in self.ex])
        return stats

    def _capture_key(self, key, issue) -> None:
        g = torch.cuda.CUDAGraph()
        if not hasattr(self, "_cap_stream"):
            self._cap_stream = torch.cuda.Stream(self.ex[0].device)
        s = self._cap_stream
        with torch.cuda.stream(s):
            g.capture_begin()
            try:
                self.stats[key] = issue(s.cuda_stream)
            finally:
                g.capture_end()
        self.graphs[key] = g
