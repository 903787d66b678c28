"""The CPU switch baseline of bench.py (SURVEY 8(d) CPU baseline (ii)) moves the right bytes.

bench.cpu_switch_copy executes the Switch Executor's weight pull plan for TP1/DP2 -> TP2/DP1 as
torch byte-slice copies and migrates KV pages with a gather/scatter per (sample, target rank);
its result must be the canonical target shards (oracle/reshard_ref.expected_shard, i.e.
tpshift/reshard.py:25-43) and every sample's KV heads of the target rank, byte for byte, or
the GB/s it reports would time the wrong copy.
"""

import numpy as np
import torch

import bench
from oracle.reshard_ref import expected_shard
from paper_2605_23945_b200.kvcache import pages_for
from paper_2605_23945_b200.models import geometry, rank_shard
from paper_2605_23945_b200.shards import arena_layout


def _geo(g):
    return dict(num_layers=g.num_layers, hidden=g.hidden, n_q=g.n_q, n_kv=g.n_kv, head_dim=g.head_dim,
                ffn=g.ffn, vocab=g.vocab, qkv_bias=g.qkv_bias, rope_theta=g.rope_theta, rms_eps=g.rms_eps)


def test_cpu_switch_copy_is_the_canonical_reshard():
    geom = geometry("mini-qwen")
    samples, ctx = 5, 130
    r = bench.cpu_switch_copy(geom, samples, ctx, threads=2, reps=1, verify=True)
    src, dsts, _, pools, new_pools, hk = r["arenas"]
    full = {}
    for (layer, fam), (off, shape) in arena_layout(geom, rank_shard(geom, 1, 0)).entries.items():
        n = int(np.prod(shape))
        t = src[off:off + 2 * n].view(torch.int16).reshape(shape)  # raw bits (NaN payloads survive)
        if fam == "w_gu":  # TP1 storage is 64-row blocks [gate c | up c]: back to [gate; up]
            blk = t.reshape(-1, 2, 64, shape[1])
            t = torch.cat([blk[:, 0].reshape(-1, shape[1]), blk[:, 1].reshape(-1, shape[1])])
        full[(layer, fam)] = t
    for rank, dst in enumerate(dsts):
        for (layer, fam), (off, shape) in arena_layout(geom, rank_shard(geom, 2, rank)).entries.items():
            want = expected_shard(_geo(geom), full, 2, rank, layer, fam).contiguous()
            got = dst[off:off + 2 * want.numel()].view(torch.int16).reshape(want.shape)
            assert torch.equal(got, want), (rank, layer, fam)
    npg = pages_for(ctx)
    for i in range(samples):
        j = i // 2
        for rank, (a, b) in enumerate(hk):
            assert torch.equal(new_pools[rank][:, :, i * npg:(i + 1) * npg],
                               pools[i % 2][:, :, j * npg:(j + 1) * npg, a:b])
    assert r["weights_bytes"] == sum(d.numel() for d in dsts) - sum(
        lay.total_bytes - sum(2 * int(np.prod(s)) for _, s in lay.entries.values())
        for lay in (arena_layout(geom, rank_shard(geom, 2, q)) for q in range(2)))
    assert r["kv_bytes"] == samples * geom.num_layers * 2 * npg * geom.n_kv * 64 * geom.head_dim * 2
    assert r["weights_gbps"] > 0 and r["kv_gbps"] > 0


def test_reference_plan_bytes_of_the_microbench_switch():
    """bench.reference_plan_bytes = the reference's priced volumes (tpshift/reshard.py:80-151):
    a TP1 -> TP2 weight reshard receives half of every layer; its KV plan counts the full hidden
    width per token (2 H bytes per layer), not the GQA heads the executor moves."""
    import argparse
    import dataclasses
    ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=8, l_max=8192, prompt_len=512, seed=4)
    spec, geom = bench.build_spec(ns, 2)
    spec = dataclasses.replace(spec, initial_tp=1, global_batch=16)
    got = bench.reference_plan_bytes(spec, 1, 2, 2, 16, 4096)
    L, H = geom.num_layers, geom.hidden
    assert got["weights"] == L * geom.layer_param_bytes // 2
    assert got["kv"] == L * 2 * 16 * 4096 * H * 2
