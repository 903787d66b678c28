"""Switch Executor: reshard a running decode from (tp, dp) to (tp', dp') on B200.

Implements the switch seam (_commit_switch, tpshift/engine.py:206-269) for
real. The reference prices -- and PAT executes -- a layer-wise All-Gather +
Slice (tpshift/reshard.py:80-151). Here every *target* rank
pulls exactly the canonical slices it owns, one-sided, from whichever rank
holds them: itself when the slice is already resident (no NVLink traffic),
otherwise a peer over NVLink (CUDA-IPC mapped pointers), with sources spread
across the old DP replicas. The result is the same canonical layout the
gather+slice would produce (rank semantics preserved), so the
transfer is copy-only and bit-exact.

Three pull plans, all pure functions of (geometry, layouts, placements):
  weights  every tensor family of every layer (QKV rows incl. the uneven
           query-head split, O columns, gate/up rows, down columns, LM-head
           vocab rows, replicated norms/embedding);
  KV       per migrated sample, layer, K|V, valid page and target kv head:
           one contiguous page_size x head_dim chunk (merge-first: samples
           land in the groups assign_merged_groups chose);
  state    token history rows (the sampler state of greedy decoding is the
           history; positions / prompt lengths are host-known).
Plans become 32-byte copy items (tps_copy_item) executed by tps_copy_items;
`verify_cover` checks that the items cover every target byte exactly once.
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass, field

import numpy as np

from .errors import PlanVerificationError
from .kvcache import PAGE, pages_for
from .models import (GLOBAL_FAMILIES, DecoderGeometry, full_shape, layer_families, rank_shard, shard_ranges)
from .shards import arena_layout

REPLICATED = ("ln1", "ln2", "ln_f", "embed")


@dataclass(frozen=True)
class Layout:
    tp: int
    world: int

    @property
    def dp(self) -> int:
        return self.world // self.tp

    def group_of(self, rank: int) -> int:
        return rank // self.tp

    def tp_rank(self, rank: int) -> int:
        return rank % self.tp

    def ranks_of_group(self, g: int) -> list[int]:
        return list(range(g * self.tp, (g + 1) * self.tp))


@dataclass
class Pieces:
    """Byte-level copy pieces: parallel int64 arrays (src_rank, src_off, dst_off, nbytes)."""

    src_rank: list = field(default_factory=list)
    src_off: list = field(default_factory=list)
    dst_off: list = field(default_factory=list)
    nbytes: list = field(default_factory=list)

    def add(self, src_rank, src_off, dst_off, nbytes):
        self.src_rank.append(np.asarray(src_rank, dtype=np.int64).ravel())
        self.src_off.append(np.asarray(src_off, dtype=np.int64).ravel())
        self.dst_off.append(np.asarray(dst_off, dtype=np.int64).ravel())
        self.nbytes.append(np.asarray(nbytes, dtype=np.int64).ravel())

    def arrays(self):
        if len(self.src_rank) > 1:  # concatenate once; later adds append to the merged arrays
            self.src_rank, self.src_off, self.dst_off, self.nbytes = (
                [np.concatenate(x)] for x in (self.src_rank, self.src_off, self.dst_off, self.nbytes))
        if not self.src_rank:
            z = np.zeros(0, dtype=np.int64)
            return z, z, z, z
        return (np.concatenate(self.src_rank), np.concatenate(self.src_off), np.concatenate(self.dst_off),
                np.concatenate(self.nbytes))


def _storage_runs(ranges):
    """[(a, b, storage_offset)] for ranges concatenated in storage order."""
    out, off = [], 0
    for a, b in ranges:
        out.append((a, b, off))
        off += b - a
    return out


def _pick_source(holders: list[int], dst_rank: int, salt: int) -> int:
    """Prefer the target rank itself (local copy); otherwise spread over the replicas."""
    if dst_rank in holders:
        return dst_rank
    return holders[(dst_rank + salt) % len(holders)]


def plan_weight_pulls(geom: DecoderGeometry, old: Layout, new: Layout, dst_rank: int) -> Pieces:
    """Pieces that fill `dst_rank`'s new arena from the old arenas (offsets are arena bytes).

    A pure function of (geometry, layouts, rank): the Cache Manager may memoise it
    (`cached_weight_pulls`). Each target run is intersected with the old tp-ranks'
    runs of the same family by bisection over the (sorted, disjoint) source runs.
    """
    new_sh = rank_shard(geom, new.tp, new.tp_rank(dst_rank))
    new_arena = arena_layout(geom, new_sh)
    old_sh = [rank_shard(geom, old.tp, r) for r in range(old.tp)]
    old_arena = [arena_layout(geom, s) for s in old_sh]
    # an old tp-rank's runs are resident on dst_rank iff dst_rank is that tp-rank in some old group
    local = [any(g * old.tp + otr == dst_rank for g in range(old.dp)) for otr in range(old.tp)]
    src_runs: dict[str, list] = {}
    pieces = Pieces()
    salt = 0
    for (layer, fam), (dst_base, dst_shape) in new_arena.entries.items():
        full = full_shape(geom, fam)
        if fam in REPLICATED:
            holders = list(range(old.world))
            src = _pick_source(holders, dst_rank, salt)
            sbase = old_arena[old.tp_rank(src)].entries[(layer, fam)][0]
            pieces.add(src, sbase, dst_base, 2 * int(np.prod(dst_shape)))
            salt += 1
            continue
        axis, dst_ranges = shard_ranges(geom, fam, new_sh)
        if fam not in src_runs:  # per family: old tp-rank runs sorted by start (c, d, storage offset)
            per = []
            for otr in range(old.tp):
                runs = sorted(_storage_runs(shard_ranges(geom, fam, old_sh[otr])[1]))
                per.append((runs, [r[1] for r in runs]))
            src_runs[fam] = per
        row_elems = full[1] if len(full) == 2 else 1
        for a, b, doff in _storage_runs(dst_ranges):
            # candidate sources: every old tp-rank run intersecting [a, b); replicated
            # KV heads appear on several tp-ranks, so sweep and take each byte once,
            # preferring a run that is resident on the target rank itself
            cands = []
            for otr, (runs, ends) in enumerate(src_runs[fam]):
                i = bisect.bisect_right(ends, a)
                while i < len(runs) and runs[i][0] < b:
                    c, d, soff = runs[i]
                    x, y = max(a, c), min(b, d)
                    if x < y:
                        cands.append((x, 0 if local[otr] else 1, y, otr, c, soff))
                    i += 1
            cands.sort()
            pos = a
            for x, _, y, otr, c, soff in cands:
                x = max(x, pos)
                if x >= y:
                    continue
                pos = y
                holders = [g * old.tp + otr for g in range(old.dp)]
                src = _pick_source(holders, dst_rank, salt)
                salt += 1
                sbase = old_arena[otr].entries[(layer, fam)][0]
                s_lo, d_lo, w = soff + (x - c), doff + (x - a), y - x
                if axis == 0 or len(full) == 1:
                    pieces.add(src, sbase + 2 * s_lo * row_elems, dst_base + 2 * d_lo * row_elems,
                               2 * w * row_elems)
                else:  # column slice of a row-major [rows][cols] tensor: one piece per row
                    rows = full[0]
                    src_ld = old_arena[otr].entries[(layer, fam)][1][1]
                    dst_ld = dst_shape[1]
                    r = np.arange(rows, dtype=np.int64)
                    pieces.add(np.full(rows, src), sbase + 2 * (r * src_ld + s_lo),
                               dst_base + 2 * (r * dst_ld + d_lo), np.full(rows, 2 * w))
    return pieces


_WEIGHT_PLANS: dict = {}


def cached_weight_pulls(geom: DecoderGeometry, old: Layout, new: Layout, dst_rank: int) -> Pieces:
    """Memoised plan_weight_pulls (plans depend only on geometry, layouts and rank)."""
    key = (geom.name, geom.num_layers, geom.hidden, old, new, dst_rank)
    if key not in _WEIGHT_PLANS:
        wp = plan_weight_pulls(geom, old, new, dst_rank)
        lay = arena_layout(geom, rank_shard(geom, new.tp, new.tp_rank(dst_rank)))
        check(verify_cover(wp, lay.total_bytes, allow_gaps=True), "weight pull plan")
        check(verify_entries(wp, lay), "weight pull plan")
        _WEIGHT_PLANS[key] = wp
    return _WEIGHT_PLANS[key]


@dataclass(frozen=True)
class KVSource:
    """Where a migrating sample lives before the switch (on every rank of its old group)."""

    old_group: int
    slot: int
    pages: tuple[int, ...]


@dataclass(frozen=True)
class KVTarget:
    slot: int
    pages: tuple[int, ...]


def kv_chunk_offset(geom: DecoderGeometry, n_kv_local: int, num_pages: int, layer: int, kv: int, page: int,
                    head: int) -> int:
    """Byte offset of a (layer, k|v, page, head) chunk in a pool [L][2][pages][nkv][64][D]."""
    chunk = PAGE * geom.head_dim * 2
    return ((((layer * 2 + kv) * num_pages + page) * n_kv_local + head) * chunk)


def plan_kv_pulls(geom: DecoderGeometry, old: Layout, new: Layout, dst_rank: int, sources: list[KVSource],
                  targets: list[KVTarget], ctx_lens: list[int], old_num_pages: int, new_num_pages: int) -> Pieces:
    """KV chunk pieces for the samples placed on dst_rank's new group (offsets are pool bytes).

    Each sample's valid pages (ceil(ctx/64)) of every layer, K and V, and every
    kv head the target rank owns are pulled from a rank of the sample's old
    group that holds that head (itself if possible).
    """
    new_sh = rank_shard(geom, new.tp, new.tp_rank(dst_rank))
    old_shards = [rank_shard(geom, old.tp, r) for r in range(old.tp)]
    L = geom.num_layers
    pieces = Pieces()
    chunk = PAGE * geom.head_dim * 2
    for src, tgt, ctx in zip(sources, targets, ctx_lens):
        npg = pages_for(ctx)
        if npg == 0:
            continue
        for h in range(*new_sh.kv_heads):
            holders = [src.old_group * old.tp + r for r in range(old.tp)
                       if old_shards[r].kv_heads[0] <= h < old_shards[r].kv_heads[1]]
            src_rank = _pick_source(holders, dst_rank, h)
            osh = old_shards[old.tp_rank(src_rank)]
            sh_ = h - osh.kv_heads[0]
            dh_ = h - new_sh.kv_heads[0]
            l = np.arange(L, dtype=np.int64)[:, None, None]
            kv = np.arange(2, dtype=np.int64)[None, :, None]
            sp = np.asarray(src.pages[:npg], dtype=np.int64)[None, None, :]
            dp = np.asarray(tgt.pages[:npg], dtype=np.int64)[None, None, :]
            soff = ((((l * 2 + kv) * old_num_pages + sp) * osh.n_kv + sh_) * chunk)
            doff = ((((l * 2 + kv) * new_num_pages + dp) * new_sh.n_kv + dh_) * chunk)
            n = soff.size
            pieces.add(np.full(n, src_rank), soff, doff, np.full(n, chunk))
    return pieces


# One KV move (tps_kv_move, include/tpshift_b200.h): a migrating sample x a run of kv heads that
# is contiguous in both pools and comes from one source rank; the device expands it into one copy
# item per (layer, k|v, valid page) reading the page tables (tps_kv_move_items).
KV_MOVE_DTYPE = np.dtype([("src_kv", "<u8"), ("src_pages", "<u8"), ("dst_pages", "<u8"),
                          ("src_num_pages", "<i4"), ("src_nkv", "<i4"), ("src_head", "<i4"),
                          ("dst_head", "<i4"), ("n_heads", "<i4"), ("n_pages", "<i4"), ("first_item", "<i8")])
assert KV_MOVE_DTYPE.itemsize == 56

# columns of a planned move (plan_kv_moves)
MV_SRC, MV_SSLOT, MV_SHEAD, MV_DSLOT, MV_DHEAD, MV_NHEADS, MV_NPAGES = range(7)

_HEAD_RUNS: dict = {}


def _head_runs(geom: DecoderGeometry, old: Layout, new: Layout, dst_rank: int, old_group: int) -> list[tuple]:
    """[(src_rank, src_head, dst_head, n_heads)] for the kv heads dst_rank owns under `new`, pulled
    from old group `old_group`: per head the same source choice as plan_kv_pulls (_pick_source,
    salt = head), consecutive heads merged while contiguous in both pools and from one rank."""
    key = (geom.name, geom.num_layers, old, new, dst_rank, old_group)
    runs = _HEAD_RUNS.get(key)
    if runs is None:
        new_sh = rank_shard(geom, new.tp, new.tp_rank(dst_rank))
        old_shards = [rank_shard(geom, old.tp, r) for r in range(old.tp)]
        runs = []
        for h in range(*new_sh.kv_heads):
            holders = [old_group * old.tp + r for r in range(old.tp)
                       if old_shards[r].kv_heads[0] <= h < old_shards[r].kv_heads[1]]
            src = _pick_source(holders, dst_rank, h)
            sh_ = h - old_shards[old.tp_rank(src)].kv_heads[0]
            dh_ = h - new_sh.kv_heads[0]
            if runs and runs[-1][0] == src and runs[-1][1] + runs[-1][3] == sh_ and runs[-1][2] + runs[-1][3] == dh_:
                runs[-1] = (src, runs[-1][1], runs[-1][2], runs[-1][3] + 1)
            else:
                runs.append((src, sh_, dh_, 1))
        _HEAD_RUNS[key] = runs
    return runs


def plan_kv_moves(geom: DecoderGeometry, old: Layout, new: Layout, dst_rank: int, old_groups, old_slots,
                  new_slots, kv_lens) -> np.ndarray:
    """KV moves of the samples placed on dst_rank's new group: int64 [n, 7] rows
    (src_rank, src_slot, src_head, dst_slot, dst_head, n_heads, n_pages).

    Covers exactly the chunks plan_kv_pulls lists (same sources; head runs merged), but
    as O(samples) rows: pages are resolved on the device from both ranks' page tables."""
    rows = []
    for og, os_, ns, n in zip(old_groups, old_slots, new_slots, kv_lens):
        npg = pages_for(int(n))
        if npg == 0:
            continue
        for src, sh_, dh_, nh in _head_runs(geom, old, new, dst_rank, int(og)):
            rows.append((src, int(os_), sh_, int(ns), dh_, nh, npg))
    return np.asarray(rows, dtype=np.int64).reshape(-1, 7)


def kv_move_bytes(geom: DecoderGeometry, moves: np.ndarray, dst_rank: int) -> tuple[int, int]:
    """(bytes pulled from peers, bytes copied locally) of planned KV moves."""
    if moves.size == 0:
        return 0, 0
    chunk = PAGE * geom.head_dim * 2
    nb = 2 * geom.num_layers * moves[:, MV_NPAGES] * moves[:, MV_NHEADS] * chunk
    remote = int(nb[moves[:, MV_SRC] != dst_rank].sum())
    return remote, int(nb.sum()) - remote


def pack_kv_moves(geom: DecoderGeometry, moves: np.ndarray, src: dict[int, dict], dst_pt: int,
                  pt_row_bytes: int) -> tuple[np.ndarray, int]:
    """Device descriptors (KV_MOVE_DTYPE) of planned moves and their total item count.
    src[rank] = {"kv": pool base, "pt": page-table base, "np": pages, "nkv": local kv heads}
    (pointers valid in this process); dst_pt = this rank's page-table base."""
    out = np.zeros(len(moves), dtype=KV_MOVE_DTYPE)
    if len(moves) == 0:
        return out, 0
    ranks = moves[:, MV_SRC]
    uniq = np.unique(ranks)
    kv = np.zeros(int(uniq.max()) + 1, dtype=np.uint64)
    pt = np.zeros_like(kv)
    npg = np.zeros(int(uniq.max()) + 1, dtype=np.int64)
    nkv = np.zeros_like(npg)
    for r in uniq:
        e = src[int(r)]
        kv[r], pt[r], npg[r], nkv[r] = e["kv"], e["pt"], e["np"], e["nkv"]
    out["src_kv"] = kv[ranks]
    out["src_pages"] = pt[ranks] + (moves[:, MV_SSLOT] * pt_row_bytes).astype(np.uint64)
    out["dst_pages"] = np.uint64(dst_pt) + (moves[:, MV_DSLOT] * pt_row_bytes).astype(np.uint64)
    out["src_num_pages"] = npg[ranks]
    out["src_nkv"] = nkv[ranks]
    out["src_head"] = moves[:, MV_SHEAD]
    out["dst_head"] = moves[:, MV_DHEAD]
    out["n_heads"] = moves[:, MV_NHEADS]
    out["n_pages"] = moves[:, MV_NPAGES]
    per = 2 * geom.num_layers * moves[:, MV_NPAGES]
    first = np.cumsum(per) - per
    out["first_item"] = first
    return out, int(per.sum())


def verify_kv_moves(moves: np.ndarray, n_kv_local: int, slots: int, expect_slots=None) -> list[str]:
    """Every (target slot, kv head) written at most once; runs inside the target's heads/slots;
    with `expect_slots`, every kv head of each of those slots (the migrated samples that have
    cached positions) written exactly once and no other slot touched."""
    if moves.size == 0:
        return ["kv heads of migrated samples not covered"] if expect_slots is not None and len(expect_slots) else []
    issues = []
    if np.any(moves[:, MV_NHEADS] <= 0) or np.any(moves[:, MV_NPAGES] <= 0):
        issues.append("empty kv move")
    if np.any(moves[:, MV_DHEAD] < 0) or np.any(moves[:, MV_DHEAD] + moves[:, MV_NHEADS] > n_kv_local):
        issues.append("kv move outside the target's kv heads")
    if np.any(moves[:, MV_DSLOT] < 0) or np.any(moves[:, MV_DSLOT] >= slots):
        issues.append("kv move outside the target's slots")
    heads = np.repeat(moves[:, MV_DSLOT] * n_kv_local + moves[:, MV_DHEAD], moves[:, MV_NHEADS])
    first = np.repeat(np.cumsum(moves[:, MV_NHEADS]) - moves[:, MV_NHEADS], moves[:, MV_NHEADS])
    heads = heads + (np.arange(heads.size) - first)
    if np.unique(heads).size != heads.size:
        issues.append("a (slot, kv head) is written twice")
    if expect_slots is not None:
        want = (np.asarray(expect_slots, dtype=np.int64)[:, None] * n_kv_local +
                np.arange(n_kv_local, dtype=np.int64)[None, :]).ravel()
        if not np.array_equal(np.sort(heads), np.sort(want)):
            issues.append("kv heads of migrated samples not covered exactly once")
    return issues


_WEIGHT_BYTES: dict = {}


def switch_bytes_per_gpu(geom: DecoderGeometry, old: Layout, new: Layout, merged, old_group, kv_len) -> dict:
    """{target rank: (bytes pulled from peers, bytes copied locally)} of a migrate switch as the
    Switch Executor runs it: the weight pulls (plan_weight_pulls, memoised), the KV moves
    (plan_kv_moves' head runs, one per (sample, kv-head run)) and the token-history rows.
    merged[g] lists the samples of new group g; old_group(s) / kv_len(s) give a sample's group
    before the switch and its cached positions."""
    chunk = PAGE * geom.head_dim * 2
    out = {}
    for r in range(new.world):
        key = (geom.name, geom.num_layers, old, new, r)
        if key not in _WEIGHT_BYTES:
            _WEIGHT_BYTES[key] = nvlink_bytes(cached_weight_pulls(geom, old, new, r), r)
        nv, loc = _WEIGHT_BYTES[key]
        g = new.group_of(r)
        for smp in (merged[g] if g < len(merged) else ()):
            og, n = int(old_group(smp)), int(kv_len(smp))
            npg = pages_for(n)
            for src, _, _, nh in _head_runs(geom, old, new, r, og):
                b = 2 * geom.num_layers * npg * nh * chunk
                if src == r:
                    loc += b
                else:
                    nv += b
            hsrc = _pick_source(old.ranks_of_group(og), r, 0)
            if hsrc == r:
                loc += 4 * (n + 1)
            else:
                nv += 4 * (n + 1)
        out[r] = (nv, loc)
    return out


def plan_history_pulls(old: Layout, dst_rank: int, sources: list[KVSource], targets: list[KVTarget],
                       lens: list[int], old_hist_ld: int, new_hist_ld: int) -> Pieces:
    """Token-history rows (prompt + generated so far) of the migrating samples."""
    pieces = Pieces()
    for src, tgt, n in zip(sources, targets, lens):
        holders = old.ranks_of_group(src.old_group)
        s = _pick_source(holders, dst_rank, 0)
        pieces.add(s, 4 * src.slot * old_hist_ld, 4 * tgt.slot * new_hist_ld, 4 * n)
    return pieces


def to_items(pieces: Pieces, src_base: dict[int, int], dst_base: int, max_chunk: int = 1 << 16) -> np.ndarray:
    """Copy items [n, 4] int64 (src_ptr, dst_ptr, bytes, 0), large pieces split to <= max_chunk."""
    sr, so, do, nb = pieces.arrays()
    if sr.size == 0:
        return np.zeros((0, 4), dtype=np.int64)
    lut = np.zeros(int(sr.max()) + 1, dtype=np.int64)
    for r in np.unique(sr):
        lut[r] = src_base[int(r)]
    bases = lut[sr]
    nsplit = (nb + max_chunk - 1) // max_chunk
    idx = np.repeat(np.arange(sr.size), nsplit)
    first = np.repeat(np.cumsum(nsplit) - nsplit, nsplit)
    k = np.arange(idx.size) - first
    off = k * max_chunk
    items = np.zeros((idx.size, 4), dtype=np.int64)
    items[:, 0] = bases[idx] + so[idx] + off
    items[:, 1] = dst_base + do[idx] + off
    items[:, 2] = np.minimum(max_chunk, nb[idx] - off)
    return items


def verify_cover(pieces: Pieces, total_bytes: int, allow_gaps: bool = False) -> list[str]:
    """Every destination byte in [0, total_bytes) written at most once (exactly once unless allow_gaps)."""
    _, _, do, nb = pieces.arrays()
    issues = []
    if do.size == 0:
        return [] if (allow_gaps or total_bytes == 0) else ["empty plan"]
    order = np.argsort(do, kind="stable")
    d, n = do[order], nb[order]
    if np.any(n <= 0):
        issues.append("non-positive piece size")
    ends = d + n
    if np.any(d[1:] < ends[:-1]):
        issues.append("overlapping destination pieces")
    if np.any(ends > total_bytes) or np.any(d < 0):
        issues.append("piece outside the destination buffer")
    if not allow_gaps:
        covered = int(n.sum())
        if covered != total_bytes:
            issues.append(f"covers {covered} of {total_bytes} bytes")
    return issues


def verify_entries(pieces: Pieces, layout) -> list[str]:
    """Every tensor of an arena layout is covered exactly: no piece crosses a tensor's payload
    bounds (or lands in the 256-B alignment padding) and each tensor's payload bytes are all
    written. With verify_cover's no-overlap check this is exactly-once coverage of every
    payload byte, which allow_gaps alone (padding is never written) cannot show."""
    _, _, do, nb = pieces.arrays()
    ents = sorted((off, 2 * int(np.prod(shape))) for off, shape in layout.entries.values())
    starts = np.array([e[0] for e in ents], dtype=np.int64)
    sizes = np.array([e[1] for e in ents], dtype=np.int64)
    idx = np.searchsorted(starts, do, side="right") - 1
    issues = []
    if np.any(idx < 0) or np.any(do + nb > starts[np.maximum(idx, 0)] + sizes[np.maximum(idx, 0)]):
        issues.append("piece outside a tensor payload")
        return issues
    got = np.bincount(idx, weights=nb.astype(np.float64), minlength=len(ents)).astype(np.int64)
    missing = int(np.count_nonzero(got != sizes))
    if missing:
        issues.append(f"{missing} tensors not covered exactly")
    return issues


def nvlink_bytes(pieces: Pieces, dst_rank: int) -> tuple[int, int]:
    """(bytes pulled from peers, bytes copied locally)."""
    sr, _, _, nb = pieces.arrays()
    remote = int(nb[sr != dst_rank].sum())
    return remote, int(nb.sum()) - remote


def check(issues: list[str], what: str) -> None:
    if issues:
        raise PlanVerificationError(f"{what}: " + "; ".join(issues))
