"""Full-size Switch Executor parity on a B200: Qwen2.5-7B weights, real pull plans.

A virtual world of `world` ranks on one device holds the Qwen2.5-7B shards of the initial
layout (seeded random, bf16); one switch runs the Switch Executor's weight / KV / history
pulls. Every new rank's weight arena must equal, byte for byte, the canonical shard of the
target layout materialised independently from the same seeded full tensors -- including
TP8's uneven 4/3 query-head split with replicated KV heads (hard part 2) --
and every migrated sample's KV pages must equal its old pages, head slice by head slice.
"""

import argparse
import dataclasses

import pytest
import torch

from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.controller import assign_merged_groups
from paper_2605_23945_b200.coordinator import B200Backend
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry, rank_shard
from paper_2605_23945_b200.shards import RankWeights
from paper_2605_23945_b200.workload import BatchStatus, Sample

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,t0,t1", [(2, 1, 2), (4, 2, 4), (8, 1, 8), (8, 8, 2)])
def test_full_size_weight_reshard_bit_exact(world, t0, t1):
    import bench
    ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=1, l_max=256, prompt_len=64, seed=4, tp_list="",
                            initial_tp=t0)
    spec, geom = bench.build_spec(ns, world)
    spec = dataclasses.replace(spec, initial_tp=t0, global_batch=world)
    be = B200Backend(spec, geom, World.virtual(world), seed=0)
    lay = be.layout
    groups = {g: [] for g in range(lay.dp)}
    for i in range(world):
        g = i % lay.dp
        slot = admit(be.group_ranks(g), i, torch.arange(spec.prompt_len, dtype=torch.int32), max_ctx=be.max_len)
        be.slot_of[i] = slot
        for r in be.group_ranks(g):
            r.slots.pos[slot] = spec.prompt_len + 10
        groups[g].append(Sample(id=i, prompt_len=spec.prompt_len, target_response_len=spec.l_max,
                                generated_len=11, intra_dp_group=g))
    merged = assign_merged_groups([BatchStatus(0, g, tuple(v)) for g, v in groups.items()], t1, spec.cluster)
    # random KV contents in the old pools; remember where each sample's pages are
    gen = torch.Generator(device="cuda").manual_seed(1)
    old = {}
    for r, rs in be.ranks.items():
        rs.kv.buf.copy_(torch.randn(rs.kv.buf.shape, generator=gen, device="cuda").to(torch.bfloat16))
        old[r] = (rs, rank_shard(geom, t0, r % t0))
    for g in range(lay.dp):  # replicated KV heads (tp > n_kv) hold identical pages, as in a run
        for h in range(geom.n_kv):
            holders = [old[g * t0 + q] for q in range(t0)
                       if old[g * t0 + q][1].kv_heads[0] <= h < old[g * t0 + q][1].kv_heads[1]]
            for rs, sh in holders[1:]:
                rs.kv.buf[:, :, :, h - sh.kv_heads[0]].copy_(
                    holders[0][0].kv.buf[:, :, :, h - holders[0][1].kv_heads[0]])
    where = {}
    for g in range(lay.dp):
        lead = be.group_ranks(g)[0]
        for slot, sid in lead.slots.sample_of.items():
            where[sid] = (g, list(lead.slots.pages[slot]))
    be._execute_switch(t1, merged)
    torch.cuda.synchronize()
    # KV: every valid page of every migrated sample, every KV head the new rank holds, equals
    # the page of a rank of the sample's old group that held that head
    kv_len = spec.prompt_len + 10  # positions < pos are cached
    npg = -(-kv_len // 64)
    for r, rs in be.ranks.items():
        nsh = rank_shard(geom, t1, r % t1)
        for slot, sid in rs.slots.sample_of.items():
            og, opages = where[sid]
            for h in range(*nsh.kv_heads):
                src = next(old[og * t0 + q] for q in range(t0)
                           if old[og * t0 + q][1].kv_heads[0] <= h < old[og * t0 + q][1].kv_heads[1])
                ors, osh = src
                for p in range(npg):
                    a = rs.kv.buf[:, :, rs.slots.pages[slot][p], h - nsh.kv_heads[0]]
                    b = ors.kv.buf[:, :, opages[p], h - osh.kv_heads[0]]
                    assert torch.equal(a, b), (t0, t1, r, sid, h, p)
    dev = torch.device("cuda:0")
    checked = set()
    for r, rs in be.ranks.items():
        tr = r % t1
        if tr in checked:  # DP replicas of one TP rank hold the same shard
            assert torch.equal(rs.weights.arena, be.ranks[tr].weights.arena)
            continue
        ref = RankWeights(geom, rank_shard(geom, t1, tr), dev).fill_random(0)
        assert torch.equal(rs.weights.arena, ref.arena), (t0, t1, r)
        checked.add(tr)
        del ref
        torch.cuda.empty_cache()
