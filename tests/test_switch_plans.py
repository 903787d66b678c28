"""CPU parity of the Switch Executor's pull plans against the oracle restatement.

Every (tp -> tp') transition over a simulated 8-GPU node: old arenas are filled
with the canonical shards of seeded full weights, the target rank's copy items
are executed on a byte-addressed CPU memory, and the result must equal the
oracle's canonical target shards byte for byte (bit-exact reshard). KV pages
and token histories are checked the same way after a merge-and-redistribute.
"""

import itertools

import numpy as np
import pytest
import torch

from oracle.decoder_ref import numpy_weights
from oracle.reshard_ref import ByteMemory, expected_shard
from paper_2605_23945_b200.models import geometry, rank_shard
from paper_2605_23945_b200.shards import arena_layout
from paper_2605_23945_b200.switch_executor import (KVSource, KVTarget, Layout, kv_chunk_offset, nvlink_bytes,
                                                   plan_history_pulls, plan_kv_pulls, plan_weight_pulls,
                                                   to_items, verify_cover)

GEOS = {name: geometry(name) for name in ("tiny", "mini-qwen")}


def geo_dict(g):
    return dict(num_layers=g.num_layers, hidden=g.hidden, n_q=g.n_q, n_kv=g.n_kv, head_dim=g.head_dim,
                ffn=g.ffn, vocab=g.vocab, qkv_bias=g.qkv_bias, rope_theta=g.rope_theta, rms_eps=g.rms_eps)


def _bytes(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).numpy().view(np.uint8).ravel()


def fill_arena(mem, base, geom, geo, full, tp, rank):
    lay = arena_layout(geom, rank_shard(geom, tp, rank))
    for (layer, fam), (off, shape) in lay.entries.items():
        blob = _bytes(expected_shard(geo, full, tp, rank, layer, fam).to(torch.bfloat16))
        mem.view(base + off, blob.size)[:] = blob


def valid_tps(geom):
    out = []
    for tp in (1, 2, 4, 8):
        try:
            geom.check_tp(tp)
            out.append(tp)
        except Exception:
            pass
    return out


@pytest.mark.parametrize("name", sorted(GEOS))
def test_weight_reshard_bit_exact_all_transitions(name):
    geom = GEOS[name]
    geo = geo_dict(geom)
    full = {k: v.to(torch.bfloat16) for k, v in numpy_weights(geo, 5).items()}
    world = 8
    tps = valid_tps(geom)
    assert len(tps) >= 3
    for t_old, t_new in itertools.product(tps, tps):
        if t_old == t_new:
            continue
        old, new = Layout(t_old, world), Layout(t_new, world)
        mem = ByteMemory()
        old_base = {}
        for r in range(world):
            lay = arena_layout(geom, rank_shard(geom, t_old, r % t_old))
            old_base[r] = mem.alloc(lay.total_bytes)
            fill_arena(mem, old_base[r], geom, geo, full, t_old, r % t_old)
        remote_total = 0
        for dst in range(world):
            lay = arena_layout(geom, rank_shard(geom, t_new, dst % t_new))
            pieces = plan_weight_pulls(geom, old, new, dst)
            payload = sum(2 * int(np.prod(s)) for _, s in lay.entries.values())
            assert verify_cover(pieces, lay.total_bytes, allow_gaps=True) == []
            assert int(pieces.arrays()[3].sum()) == payload
            base = mem.alloc(lay.total_bytes)
            mem.execute(to_items(pieces, old_base, base, max_chunk=4096))
            for (layer, fam), (off, shape) in lay.entries.items():
                want = _bytes(expected_shard(geo, full, t_new, dst % t_new, layer, fam).to(torch.bfloat16))
                got = mem.view(base + off, want.size)
                assert np.array_equal(got, want), (t_old, t_new, dst, layer, fam)
            remote, local = nvlink_bytes(pieces, dst)
            remote_total += remote
            if t_old == 1:  # every target slice is already resident: zero NVLink bytes
                assert remote == 0
        if t_old < t_new and t_new % t_old == 0 and t_old > 1:
            assert remote_total > 0


def test_kv_and_history_migration_bit_exact():
    geom = GEOS["mini-qwen"]
    world, L, D = 8, geom.num_layers, geom.head_dim
    rng = np.random.default_rng(0)
    for t_old, t_new in [(1, 2), (1, 8), (2, 8), (4, 2), (2, 4), (8, 1)]:
        old, new = Layout(t_old, world), Layout(t_new, world)
        n_samples = 5
        ctx = [int(x) for x in rng.integers(1, 300, n_samples)]
        old_group = [int(x) for x in rng.integers(0, old.dp, n_samples)]
        num_pages_old, num_pages_new, max_pages = 64, 64, 8
        hist_ld = 512
        # logical truth: kv[(sample, layer, kvsel, head)] -> [ctx, D] bf16 bytes ; history[sample] -> ints
        truth = {}
        mem = ByteMemory()
        pool_base, hist_base, src_desc = {}, {}, []
        old_pages = {}
        for r in range(world):
            sh = rank_shard(geom, t_old, r % t_old)
            pool_base[r] = mem.alloc(L * 2 * num_pages_old * sh.n_kv * 64 * D * 2)
            hist_base[r] = mem.alloc(16 * hist_ld * 4)
        perm = rng.permutation(num_pages_old)  # disjoint page sets per sample
        for i in range(n_samples):
            pages = tuple(int(p) for p in perm[i * max_pages:(i + 1) * max_pages])
            old_pages[i] = pages
            slot = 3 + i
            src_desc.append(KVSource(old_group=old_group[i], slot=slot, pages=pages))
            hist = rng.integers(0, 1 << 20, ctx[i]).astype(np.int32)
            truth[("h", i)] = hist
            for h in range(geom.n_kv):
                for l in range(L):
                    for kv in range(2):
                        truth[(i, l, kv, h)] = rng.integers(0, 256, (ctx[i], D * 2)).astype(np.uint8)
            for r in old.ranks_of_group(old_group[i]):
                sh = rank_shard(geom, t_old, r % t_old)
                mem.view(hist_base[r] + 4 * slot * hist_ld, 4 * ctx[i])[:] = hist.view(np.uint8)
                for h in range(*sh.kv_heads):
                    for l in range(L):
                        for kv in range(2):
                            tok = truth[(i, l, kv, h)]
                            for p in range((ctx[i] + 63) // 64):
                                off = kv_chunk_offset(geom, sh.n_kv, num_pages_old, l, kv, pages[p],
                                                      h - sh.kv_heads[0])
                                rows = tok[p * 64:(p + 1) * 64]
                                mem.view(pool_base[r] + off, rows.size)[:] = rows.ravel()
        # merge: samples spread over the new groups round-robin
        placement = {g: [i for i in range(n_samples) if i % new.dp == g] for g in range(new.dp)}
        for dst in range(world):
            g = new.group_of(dst)
            mine = placement[g]
            sh = rank_shard(geom, t_new, dst % t_new)
            tgts = [KVTarget(slot=j, pages=tuple(range(j * max_pages, (j + 1) * max_pages))) for j in range(len(mine))]
            srcs = [src_desc[i] for i in mine]
            kp = plan_kv_pulls(geom, old, new, dst, srcs, tgts, [ctx[i] for i in mine], num_pages_old, num_pages_new)
            hp = plan_history_pulls(old, dst, srcs, tgts, [ctx[i] for i in mine], hist_ld, hist_ld)
            pool_sz = L * 2 * num_pages_new * sh.n_kv * 64 * D * 2
            assert verify_cover(kp, pool_sz, allow_gaps=True) == []
            nb = mem.alloc(pool_sz)
            hb = mem.alloc(16 * hist_ld * 4)
            mem.execute(to_items(kp, pool_base, nb))
            mem.execute(to_items(hp, hist_base, hb))
            for j, i in enumerate(mine):
                got_hist = mem.view(hb + 4 * j * hist_ld, 4 * ctx[i]).view(np.int32)
                assert np.array_equal(got_hist, truth[("h", i)])
                for h in range(*sh.kv_heads):
                    for l in range(L):
                        for kv in range(2):
                            tok = truth[(i, l, kv, h)]
                            for p in range((ctx[i] + 63) // 64):
                                off = kv_chunk_offset(geom, sh.n_kv, num_pages_new, l, kv, tgts[j].pages[p],
                                                      h - sh.kv_heads[0])
                                n = min(64, ctx[i] - p * 64)
                                got = mem.view(nb + off, n * D * 2).reshape(n, D * 2)
                                assert np.array_equal(got, tok[p * 64:p * 64 + n]), (t_old, t_new, i, l, kv, h, p)


def test_prefill_group_table():
    """Host side of the grouped prefill attention: each sample's rows in chunk order, cut at
    `gp` positions, padding rows in no group, every row in exactly one group."""
    import numpy as np
    from paper_2605_23945_b200.executor import prefill_groups
    rs = np.array([0, 1, 2, 0, 1, 2, 0, 1, -1, 0, 0, 0, 5])
    rows, n = prefill_groups(rs, 3)
    assert n.tolist()[:6] == [3, 3, 2, 3, 1, 0]
    assert rows[0, :3].tolist() == [0, 3, 6] and rows[3, :3].tolist() == [9, 10, 11] and rows[4, 0] == 12
    got = sorted(int(r) for g in range(len(n)) for r in rows[g, :n[g]])
    assert got == [i for i in range(len(rs)) if rs[i] >= 0]
    for g in range(len(n)):
        assert len({int(rs[r]) for r in rows[g, :n[g]]}) <= 1


def test_weight_plan_entry_coverage_check():
    """verify_entries accepts every real weight plan and rejects a plan missing one piece or
    writing into alignment padding (the runtime check cached_weight_pulls applies)."""
    from paper_2605_23945_b200.switch_executor import Pieces, cached_weight_pulls, verify_entries
    geom = geometry("mini-qwen")
    old, new = Layout(1, 4), Layout(4, 4)
    for r in range(4):
        wp = cached_weight_pulls(geom, old, new, r)
        lay = arena_layout(geom, rank_shard(geom, 4, r))
        assert verify_entries(wp, lay) == []
        sr, so, do, nb = wp.arrays()
        cut = Pieces()
        cut.add(sr[1:], so[1:], do[1:], nb[1:])
        assert verify_entries(cut, lay)
        off, shape = lay.entries[(-1, "ln_f")]
        pad = Pieces()
        pad.add(sr, so, do, nb)
        pad.add(np.array([0]), np.array([0]), np.array([off + 2 * int(np.prod(shape))]), np.array([2]))
        assert verify_entries(pad, lay)


@pytest.mark.parametrize("gname", ["mini-qwen", "tiny", "mini-llama"])
def test_kv_moves_match_the_chunk_plan_and_migrate_bit_exact(gname):
    """The O(samples) KV moves (expanded from page tables, as tps_kv_move_items does on the
    device) copy exactly the chunks plan_kv_pulls lists, and the migrated pages are bit-exact --
    with KV heads replicated (tp > n_kv: mini-qwen, tiny) and split (mini-llama)."""
    from oracle.reshard_ref import expand_kv_moves
    from paper_2605_23945_b200.models import geometry as _geometry
    from paper_2605_23945_b200.switch_executor import (kv_move_bytes, pack_kv_moves, plan_kv_moves,
                                                       verify_kv_moves)
    geom = _geometry(gname)
    world, L, D = 8, geom.num_layers, geom.head_dim
    chunk = 64 * D * 2
    rng = np.random.default_rng(1)
    for t_old, t_new in [(1, 2), (1, 8), (2, 8), (4, 2), (2, 4), (8, 1), (4, 8)]:
        try:
            geom.check_tp(t_old)
            geom.check_tp(t_new)
        except Exception:
            continue
        old, new = Layout(t_old, world), Layout(t_new, world)
        n_samples, P, npg_old, npg_new = 6, 8, 64, 80
        ctx = [int(x) for x in rng.integers(1, 400, n_samples)]
        old_group = [int(x) for x in rng.integers(0, old.dp, n_samples)]
        old_slot = [2 + i for i in range(n_samples)]
        mem = ByteMemory()
        src = {}
        perm = rng.permutation(npg_old)
        for r in range(world):
            sh = rank_shard(geom, t_old, r % t_old)
            base = mem.alloc(L * 2 * npg_old * sh.n_kv * chunk)
            mem.view(base, L * 2 * npg_old * sh.n_kv * chunk)[:] = rng.integers(0, 256, L * 2 * npg_old * sh.n_kv * chunk,
                                                                                 dtype=np.uint8)
            pt = mem.alloc(16 * P * 4)
            for i in range(n_samples):
                mem.view(pt + 4 * P * old_slot[i], 4 * P)[:] = perm[i * P:(i + 1) * P].astype(np.int32).view(np.uint8)
            src[r] = {"kv": base, "pt": pt, "np": npg_old, "nkv": sh.n_kv}
        placement = {g: [i for i in range(n_samples) if i % new.dp == g] for g in range(new.dp)}
        for dst in range(world):
            mine = placement[new.group_of(dst)]
            sh = rank_shard(geom, t_new, dst % t_new)
            new_slot = [5 + j for j in range(len(mine))]
            pt_new = mem.alloc(16 * P * 4)
            tgt_pages = {}
            dperm = rng.permutation(npg_new).astype(np.int32)  # disjoint page sets per sample
            for j, i in enumerate(mine):
                pages = dperm[j * P:(j + 1) * P]
                tgt_pages[i] = pages
                mem.view(pt_new + 4 * P * new_slot[j], 4 * P)[:] = pages.view(np.uint8)
            moves = plan_kv_moves(geom, old, new, dst, [old_group[i] for i in mine], [old_slot[i] for i in mine],
                                  new_slot, [ctx[i] for i in mine])
            assert verify_kv_moves(moves, sh.n_kv, 16, new_slot) == []
            if len(moves) > 1:  # a dropped run is caught
                assert verify_kv_moves(moves[1:], sh.n_kv, 16, new_slot)
            packed, n_items = pack_kv_moves(geom, moves, src, pt_new, 4 * P)
            pool = mem.alloc(L * 2 * npg_new * sh.n_kv * chunk)
            items = expand_kv_moves(mem, packed, pool, npg_new, sh.n_kv, L, chunk)
            assert len(items) == n_items
            # same bytes, same sources as the per-chunk plan
            srcs = [KVSource(old_group=old_group[i], slot=old_slot[i], pages=tuple(int(p) for p in perm[i * P:(i + 1) * P]))
                    for i in mine]
            tgts = [KVTarget(slot=new_slot[j], pages=tuple(int(p) for p in tgt_pages[i])) for j, i in enumerate(mine)]
            kp = plan_kv_pulls(geom, old, new, dst, srcs, tgts, [ctx[i] for i in mine], npg_old, npg_new)
            ref = to_items(kp, {r: src[r]["kv"] for r in src}, pool)
            split = []
            for s, d, n, _ in items:
                for k in range(n // chunk):
                    split.append((s + k * chunk, d + k * chunk, chunk, 0))
            assert sorted(map(tuple, ref.tolist())) == sorted(split)
            assert sum(kv_move_bytes(geom, moves, dst)) == int(ref[:, 2].sum()) if len(ref) else True
            assert kv_move_bytes(geom, moves, dst) == nvlink_bytes(kp, dst)
            mem.execute(items)
            for s, d, n, _ in ref:
                assert np.array_equal(mem.view(int(s), int(n)), mem.view(int(d), int(n)))


def test_kv_move_plan_rejects_double_writes():
    from paper_2605_23945_b200.switch_executor import verify_kv_moves
    ok = np.array([[0, 1, 0, 3, 0, 2, 4], [1, 2, 0, 4, 0, 2, 4]], dtype=np.int64)
    assert verify_kv_moves(ok, 2, 8) == []
    dup = np.array([[0, 1, 0, 3, 0, 2, 4], [1, 2, 1, 3, 1, 1, 4]], dtype=np.int64)
    assert verify_kv_moves(dup, 2, 8)
    assert verify_kv_moves(np.array([[0, 1, 0, 9, 0, 1, 4]], dtype=np.int64), 2, 8)


def test_kv_moves_edge_cases():
    """Empty target groups, samples with no cached positions yet, and one-position contexts."""
    from paper_2605_23945_b200.switch_executor import (kv_move_bytes, pack_kv_moves, plan_kv_moves,
                                                       verify_kv_moves)
    geom = GEOS["mini-qwen"]
    old, new = Layout(1, 4), Layout(2, 4)
    empty = plan_kv_moves(geom, old, new, 0, [], [], [], [])
    assert empty.shape == (0, 7) and verify_kv_moves(empty, 1, 4) == []
    assert kv_move_bytes(geom, empty, 0) == (0, 0)
    packed, n = pack_kv_moves(geom, empty, {}, 0, 64)
    assert n == 0 and len(packed) == 0
    mv = plan_kv_moves(geom, old, new, 1, [2, 3], [0, 1], [0, 1], [0, 1])  # kv_len 0 -> no pages
    assert mv.shape[0] == 1 and int(mv[0, 6]) == 1                         # kv_len 1 -> one page
    chunk = 64 * geom.head_dim * 2
    nb = sum(kv_move_bytes(geom, mv, 1))
    assert nb == 2 * geom.num_layers * int(mv[0, 5]) * chunk


def test_weight_plan_identity_transition_is_all_local():
    """tp -> the same tp (a regroup): every byte is copied locally, none pulled."""
    geom = GEOS["mini-qwen"]
    for tp in (1, 2):
        lay = Layout(tp, 4)
        for r in range(4):
            nv, loc = nvlink_bytes(plan_weight_pulls(geom, lay, lay, r), r)
            assert nv == 0 and loc == arena_layout(geom, rank_shard(geom, tp, r % tp)).total_bytes - \
                _padding(geom, tp, r % tp)


def _padding(geom, tp, r):
    lay = arena_layout(geom, rank_shard(geom, tp, r))
    payload = sum(2 * int(np.prod(shape)) for _, shape in lay.entries.values())
    return lay.total_bytes - payload
