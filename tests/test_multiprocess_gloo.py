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
