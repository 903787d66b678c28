"""World-size-2 `gloo` tests of the multi-process host logic (no GPU needed).

One process per GPU runs the Global Coordinator SPMD: every rank evaluates
Algorithm 1 on the same node state and must reach identical decisions without
exchanging control messages; at a switch each rank plans only its own pulls,
and the union of the per-rank plans must cover every target shard exactly
once, byte-exact against the oracle (checked on rank 0 after a gather).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_23945_b200.cache_manager import World
        from paper_2605_23945_b200.config import build_scenario, load_config
        from paper_2605_23945_b200.engine import run
        from paper_2605_23945_b200.models import geometry
        from paper_2605_23945_b200.switch_executor import Layout, plan_weight_pulls

        w = World(gpus=world, local_ranks=[rank], devices={rank: torch.device("cpu")}, distributed=True)
        # (1) SPMD decisions: identical switch sequences on every rank
        rep = run(build_scenario(load_config("paper_a40"), l_max=12288, seed=3))
        sw = [(s["round"], s["from_tp"], s["to_tp"]) for nr in rep.node_reports for s in nr["switches"]]
        all_sw = w.allgather(sw)
        # (2) per-rank weight pull plans of an 8-GPU node, ranks split across the 2 processes
        geom = geometry("mini-qwen")
        plans = {}
        for dst in range(rank, 8, world):
            p = plan_weight_pulls(geom, Layout(2, 8), Layout(8, 8), dst)
            plans[dst] = [a.tolist() for a in p.arrays()]
        gathered = w.allgather(plans)
        w.barrier()
        q.put((rank, all_sw, gathered if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_spmd_decisions_and_distributed_pull_plans():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    by_rank = {r: (sw, g) for r, sw, g in out}
    sw0 = by_rank[0][0]
    assert sw0[0] == sw0[1], "ranks reached different switch decisions"
    assert len(sw0[0]) >= 1
    # union of both processes' plans covers every target arena exactly, byte-exact vs the oracle
    import numpy as np

    from oracle.decoder_ref import numpy_weights
    from oracle.reshard_ref import ByteMemory, expected_shard
    from paper_2605_23945_b200.models import geometry, rank_shard
    from paper_2605_23945_b200.shards import arena_layout
    from paper_2605_23945_b200.switch_executor import Pieces, to_items, verify_cover

    geom = geometry("mini-qwen")
    geo = dict(num_layers=geom.num_layers, hidden=geom.hidden, n_q=geom.n_q, n_kv=geom.n_kv,
               head_dim=geom.head_dim, ffn=geom.ffn, vocab=geom.vocab, qkv_bias=geom.qkv_bias,
               rope_theta=geom.rope_theta, rms_eps=geom.rms_eps)
    full = {k: v.to(torch.bfloat16) for k, v in numpy_weights(geo, 9).items()}
    mem = ByteMemory()
    old = {}
    for r in range(8):
        lay = arena_layout(geom, rank_shard(geom, 2, r % 2))
        old[r] = mem.alloc(lay.total_bytes)
        for (layer, fam), (off, shape) in lay.entries.items():
            blob = expected_shard(geo, full, 2, r % 2, layer, fam).contiguous().view(torch.int16).numpy()
            blob = blob.view(np.uint8).ravel()
            mem.view(old[r] + off, blob.size)[:] = blob
    merged = {}
    for part in by_rank[0][1]:
        merged.update(part)
    assert sorted(merged) == list(range(8))
    for dst, arrs in merged.items():
        p = Pieces()
        p.add(*[np.asarray(a, dtype=np.int64) for a in arrs])
        lay = arena_layout(geom, rank_shard(geom, 8, dst))
        assert verify_cover(p, lay.total_bytes, allow_gaps=True) == []
        base = mem.alloc(lay.total_bytes)
        mem.execute(to_items(p, old, base))
        for (layer, fam), (off, shape) in lay.entries.items():
            want = expected_shard(geo, full, 8, dst, layer, fam).contiguous().view(torch.int16).numpy()
            want = want.view(np.uint8).ravel()
            assert np.array_equal(mem.view(base + off, want.size), want), (dst, layer, fam)


def _kv_worker(rank, world, port, q):
    """Each process owns ranks {rank, rank + world, ...} of an 8-GPU node. As in
    B200Backend._execute_switch: every process reports where its groups' samples sit, the
    reports are all-gathered, and each process plans the KV moves of its own target ranks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_23945_b200.cache_manager import World
        from paper_2605_23945_b200.models import geometry
        from paper_2605_23945_b200.switch_executor import Layout, plan_kv_moves

        w = World(gpus=world, local_ranks=[rank], devices={rank: torch.device("cpu")}, distributed=True)
        geom = geometry("mini-qwen")
        old, new = Layout(2, 8), Layout(8, 8)
        mine = [r for r in range(8) if r % world == rank]
        # old placement: sample i in old group i % 4 at slot 1 + i // 4; the lead rank of a group
        # reports it (the group's ranks live in different processes)
        here = {i: (i % 4, 1 + i // 4) for i in range(10) if (i % 4) * old.tp in mine}
        where = {}
        for part in w.allgather(here):
            where.update(part)
        plans = {}
        for dst in mine:
            ids = list(range(10))  # TP8/DP1: every sample lands on the one group
            moves = plan_kv_moves(geom, old, new, dst, [where[i][0] for i in ids], [where[i][1] for i in ids],
                                  [2 + i for i in ids], [37 * i + 5 for i in ids])
            plans[dst] = moves.tolist()
        q.put((rank, w.allgather(plans)))
    finally:
        dist.destroy_process_group()


def test_distributed_kv_move_plans_cover_every_head_once():
    """The union of the per-process KV-move plans (each process planning only its target ranks
    from the all-gathered placement) moves every (sample, kv head) each target rank owns exactly
    once, from a rank of the sample's old group that holds that head."""
    import numpy as np

    from paper_2605_23945_b200.models import geometry, rank_shard
    from paper_2605_23945_b200.switch_executor import Layout, plan_kv_moves
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kv_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for part in out[0][1]:
        merged.update(part)
    assert sorted(merged) == list(range(8))
    geom = geometry("mini-qwen")
    old, new = Layout(2, 8), Layout(8, 8)
    for dst, rows in merged.items():
        sh = rank_shard(geom, 8, dst)
        got = set()
        for src, sslot, shead, dslot, dhead, nh, npg in rows:
            assert src // old.tp == (dslot - 2) % 4 and sslot == 1 + (dslot - 2) // 4  # the sample's old group / slot
            osh = rank_shard(geom, old.tp, src % old.tp)
            for h in range(nh):
                gh = osh.kv_heads[0] + shead + h
                assert gh == sh.kv_heads[0] + dhead + h  # same global kv head on both sides
                got.add((dslot, dhead + h))
            assert npg == -(-(37 * (dslot - 2) + 5) // 64)
        assert got == {(2 + i, h) for i in range(10) for h in range(sh.n_kv)}
        # the same plan a single process makes
        ids = list(range(10))
        ref = plan_kv_moves(geom, old, new, dst, [i % 4 for i in ids], [1 + i // 4 for i in ids],
                            [2 + i for i in ids], [37 * i + 5 for i in ids])
        assert np.array_equal(np.asarray(rows, dtype=np.int64).reshape(-1, 7), ref)
