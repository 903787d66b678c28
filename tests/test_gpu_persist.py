"""The persistent one-launch decode step (csrc/persist.cu) against the per-kernel step and
itself: determinism, CUDA-graph replay, alternation with the per-kernel / counter / prefill
protocols inside one TP layout, and the group epoch / phase counters it must keep in step.

Numerical parity with the CPU oracle is covered where the decode tests run B <= 16 (they take
the persistent path by default): tests/test_gpu_decode.py (mini geometries, TP1..8) and
tests/test_gpu_decode_fullshape.py (true per-layer shapes, 8K/16K contexts, both paths).
"""

import pytest
import torch

from paper_2605_23945_b200.group import admit, build_group, last_logits
from paper_2605_23945_b200.models import geometry

pytestmark = pytest.mark.gpu


def _group(name, tp, B, persist, graphs=True, max_len=160, seed=7):
    geom = geometry(name)
    ranks, runner = build_group(geom, tp, max_batch=max(B, 8), num_slots=B + 2, max_len=max_len, seed=seed,
                                use_graphs=graphs)
    for r in ranks:
        r.executor.use_persist = persist
    gen = torch.Generator().manual_seed(B * 31 + tp)
    prompts = torch.randint(0, geom.vocab, (B, 6), generator=gen).tolist()
    slots = [admit(ranks, i, p, max_ctx=len(p) + 40) for i, p in enumerate(prompts)]
    bk = ranks[0].executor.bucket(B)
    runner.set_rows(bk, slots)
    return ranks, runner, slots, bk


@pytest.mark.parametrize("name,tp,B", [("mini-qwen", 1, 1), ("mini-qwen", 2, 3), ("mini-qwen", 4, 8),
                                       ("mini-llama", 8, 2), ("mini-qwen32", 8, 12), ("mini-llama", 1, 16),
                                       ("mini-qwen", 2, 4), ("mini-llama", 4, 1)])
def test_persist_matches_per_kernel_step(name, tp, B):
    """Same weights and prompts: logits within the decode tolerance, greedy tokens equal
    wherever the per-kernel step's top-2 margin exceeds 0.1."""
    out = {}
    for persist in (True, False):
        ranks, runner, slots, bk = _group(name, tp, B, persist, graphs=False)
        assert runner.persist_ok(bk) == persist
        lg = []
        for _ in range(12):
            runner.step(bk, 1)
            lg.append(last_logits(ranks)[:B].cpu())
        torch.cuda.synchronize()
        out[persist] = (torch.stack(lg), ranks[0].slots.history[slots].cpu())
    (lp, hp), (lk, hk) = out[True], out[False]
    # teacher forcing differs once a token differs; compare up to the first divergence
    assert torch.equal(hp[:, :6], hk[:, :6])
    for t in range(12):
        d = float((lp[t] - lk[t]).abs().max())
        assert d <= 0.05, (t, d)
        top2 = lk[t].topk(2, dim=1).values
        sure = (top2[:, 0] - top2[:, 1]) > 0.1
        if t >= 5:
            pos = t + 1
            assert torch.equal(hp[sure, pos], hk[sure, pos]), t
            if not torch.equal(hp[:, pos], hk[:, pos]):
                break


@pytest.mark.parametrize("name,tp,B", [("mini-qwen", 1, 4), ("mini-qwen", 2, 16), ("mini-llama", 8, 1),
                                       ("mini-qwen", 4, 2), ("mini-qwen32", 2, 8)])
def test_persist_graph_replay_equals_eager_and_is_deterministic(name, tp, B):
    hist = []
    for graphs in (False, True, True):
        ranks, runner, slots, bk = _group(name, tp, B, True, graphs=graphs)
        runner.step(bk, 1)
        if graphs:
            runner.capture(bk)
        runner.step(bk, 20)
        torch.cuda.synchronize()
        hist.append(ranks[0].slots.history[slots].cpu())
        assert runner.kernels_per_step(bk) == 1
    assert torch.equal(hist[0], hist[1]) and torch.equal(hist[1], hist[2])


def test_persist_alternates_with_per_kernel_and_counter_protocols_tp2():
    """One TP2 layout runs persistent steps (B <= 16), LL per-kernel steps (B 24..64), counter
    steps (B > 64) and a chunked prefill in any order: the group epoch and every phase counter
    stay at epoch * tp, no wait can deadlock, logits stay finite."""
    geom = geometry("mini-qwen")
    ranks, runner = build_group(geom, 2, max_batch=96, num_slots=96, max_len=96, seed=4)
    for r in ranks:
        r.executor.prefill_rows = 0
        r.executor.use_persist = True
    slots = [admit(ranks, i, [1 + i % 50, 2, 3], max_ctx=64) for i in range(80)]
    for B, n in ((4, 3), (16, 2), (80, 2), (1, 2), (40, 1), (96, 1), (8, 3), (64, 1), (2, 2)):
        bk = ranks[0].executor.bucket(B)
        runner.set_rows(bk, slots[:min(B, 80)])
        runner.step(bk, n)
        lg = last_logits(ranks)
        torch.cuda.synchronize()
        assert torch.isfinite(lg[:min(B, 80)]).all(), B
    for r in ranks:
        cm = r.executor.comm
        ep = int(cm.epoch.item())
        L = geom.num_layers
        assert cm.ctr[:2 * L + 1].tolist() == [(ep - 1) * 2] * (2 * L + 1)


def test_persist_loopback_rank_runs():
    """The profiler's timing harness (one TP8 rank playing every peer) takes the persistent
    path: LL pushes into its own tp slots, argmax candidates likewise."""
    from paper_2605_23945_b200.profiler import loopback_rank
    geom = geometry("mini-llama")
    r, runner = loopback_rank(geom, 8, 4, 4, 256, 4 * 5)
    r.executor.use_persist = True
    slots = [admit([r], i, [1, 2, 3], max_ctx=200) for i in range(4)]
    runner.set_rows(4, slots)
    assert runner.persist_ok(4)
    runner.step(4, 1)
    runner.capture(4)
    runner.step(4, 10)
    torch.cuda.synchronize()
    assert int(r.slots.pos[slots[0]]) == 11
