"""Kernel-level numerics of libtpshift_b200 on a B200 against plain PyTorch fp32 references.

Tolerances: projections accumulate bf16 x bf16 in fp32 on the tensor cores, so
they are compared with a torch fp32 matmul of the same bf16 inputs at
|d| <= 1e-3 * sqrt(K) * max|ref| relative slack; copies are bit-exact.
"""

import ctypes
import math

import pytest
import torch

from paper_2605_23945_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    nat.init_device(0)


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("n,k,b", [
    (128, 64, 1), (384, 256, 5), (4736, 3584, 16), (1000, 104, 17), (256, 4096, 64),
    (3584, 18944, 33), (768, 512, 100), (512, 1024, 256), (8192, 256, 2),
    (3584, 512, 300), (640, 1024, 1000), (4736, 3584, 512)])  # > 256 rows: activation tiles
def test_linear_matches_fp32(n, k, b):
    torch.manual_seed(n + k + b)
    w = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    x = torch.randn(b + 3, k, device="cuda").bfloat16()  # extra rows are never read
    ref = x[:b].float() @ w.float().T
    lib = nat.lib()
    for splits in sorted({1, lib.tps_linear_splits(n, k, b), min(3, (k + 63) // 64)}):
        out = torch.full((splits, b, n), float("nan"), device="cuda")
        nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), b, x.shape[0], k, out.data_ptr(),
                                 splits, _stream()))
        got = out.sum(0)
        torch.cuda.synchronize()
        tol = 2e-3 * math.sqrt(k) * 0.05 * 4 + 1e-4
        assert torch.isfinite(got).all()
        assert (got - ref).abs().max().item() <= tol, (splits, (got - ref).abs().max().item())


def test_linear_rejects_bad_args():
    lib = nat.lib()
    from paper_2605_23945_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        nat.check(lib.tps_linear(0, 128, 64, 64, 0, 1, 1, 64, 0, 1, _stream()))
    w = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(1, 300, 128, device="cuda")
    with pytest.raises(ConfigError):  # fewer activation rows than the batch
        nat.check(lib.tps_linear(w.data_ptr(), 128, 64, 64, w.data_ptr(), 300, 200, 64, out.data_ptr(), 1,
                                 _stream()))
    with pytest.raises(ConfigError):  # more splits than 64-wide K chunks
        nat.check(lib.tps_linear(w.data_ptr(), 128, 64, 64, w.data_ptr(), 1, 1, 64, out.data_ptr(), 2,
                                 _stream()))


def _ref_attention(q, kc, vc, page_table, pos, G):
    """q [B, nq, D]; kc/vc [pages, nkv, 64, D]; returns [B, nq, D] fp32."""
    B, nq, D = q.shape
    out = torch.zeros(B, nq, D)
    for b in range(B):
        ctx = pos[b] + 1
        pages = page_table[b][: (ctx + 63) // 64]
        K = torch.cat([kc[p] for p in pages], dim=1)[:, :ctx].float()  # [nkv, T, D]
        V = torch.cat([vc[p] for p in pages], dim=1)[:, :ctx].float()
        for h in range(nq):
            kvh = h // G
            s = (K[kvh] @ q[b, h].float()) / math.sqrt(D)
            p = torch.softmax(s, dim=0)
            out[b, h] = p @ V[kvh]
    return out


@pytest.mark.parametrize("D,nq,nkv,ctxs", [
    (128, 7, 1, [1, 64, 65, 300]), (128, 28, 4, [5000, 17]), (64, 4, 2, [130, 1]),
    (128, 4, 1, [2049]), (128, 16, 1, [100, 1000])])
def test_paged_attention_matches_fp32(D, nq, nkv, ctxs):
    """Cluster form (nsplit -1, DSMEM merge), page-balanced schedule (nsplit 0) and fixed split
    counts (in-kernel and combine merge)."""
    torch.manual_seed(D + nq + len(ctxs))
    B = len(ctxs)
    max_pages = max((c + 63) // 64 for c in ctxs) + 1
    num_pages = B * max_pages + 3
    kc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    vc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    perm = torch.randperm(num_pages)[: B * max_pages].view(B, max_pages).int()
    page_table = perm.cuda()
    row_slot = torch.arange(B, dtype=torch.int32, device="cuda")
    pos = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32, device="cuda")
    q = torch.randn(B, nq, D, device="cuda").bfloat16()
    lib = nat.lib()
    ctr = torch.zeros(B * nkv, dtype=torch.int32, device="cuda")
    for nsplit in (-1, 0, 1, lib.tps_attn_splits(B, nkv, max_pages), 7):
        ws = lib.tps_attn_workspace(B, nq, D, nsplit)
        pm = torch.empty(ws // D, device="cuda")
        pl = torch.empty_like(pm)
        po = torch.empty(ws, device="cuda")
        out = torch.empty(B, nq, D, device="cuda", dtype=torch.bfloat16)
        nat.check(lib.tps_paged_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), row_slot.data_ptr(),
                                          pos.data_ptr(), None, page_table.data_ptr(), max_pages, B, nq, nkv, D,
                                          nsplit, pm.data_ptr(), pl.data_ptr(), po.data_ptr(), ctr.data_ptr(), out.data_ptr(), None, 0, 0, None, None, None,
                                          _stream()))
        torch.cuda.synchronize()
        ref = _ref_attention(q.cpu(), kc.cpu(), vc.cpu(), perm.tolist(), [c - 1 for c in ctxs], nq // nkv)
        err = (out.float().cpu() - ref).abs().max().item()
        # P is rounded to bf16 before the PV product; outputs are O(1)
        assert err < 2e-2, (nsplit, err)
        assert int(ctr.sum()) == 0  # merge counters re-armed by the last CTA


@pytest.mark.parametrize("nsplit", [0, 3])
def test_padding_rows_are_inert(nsplit):
    D, nq, nkv = 128, 4, 1
    kc = torch.randn(4, nkv, 64, D, device="cuda").bfloat16()
    vc = torch.randn_like(kc)
    page_table = torch.zeros(1, 2, dtype=torch.int32, device="cuda")
    row_slot = torch.tensor([-1, 0], dtype=torch.int32, device="cuda")
    pos = torch.tensor([10], dtype=torch.int32, device="cuda")
    q = torch.randn(2, nq, D, device="cuda").bfloat16()
    ws = nat.lib().tps_attn_workspace(2, nq, D, nsplit)
    pm = torch.empty(ws // D, device="cuda")
    pl, po = torch.empty_like(pm), torch.empty(ws, device="cuda")
    out = torch.full((2, nq, D), 7.0, device="cuda", dtype=torch.bfloat16)
    ctr = torch.zeros(2 * nkv, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().tps_paged_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), row_slot.data_ptr(),
                                            pos.data_ptr(), None, page_table.data_ptr(), 2, 2, nq, nkv, D, nsplit,
                                            pm.data_ptr(), pl.data_ptr(), po.data_ptr(), ctr.data_ptr(), out.data_ptr(), None, 0, 0, None, None, None,
                                            _stream()))
    torch.cuda.synchronize()
    assert (out[0] == 0).all()
    assert torch.isfinite(out[1].float()).all()


@pytest.mark.parametrize("B,max_ctx,prefill", [(200, 3000, False), (3, 20000, False), (512, 700, True)])
def test_balanced_attention_ragged(B, max_ctx, prefill):
    """Page-balanced schedule on ragged batches: segments cut across many CTAs, one
    very long row next to short ones, and the prefill form (row_pos, 512 rows)."""
    torch.manual_seed(B)
    D, nq, nkv = 128, 28, 4
    lib = nat.lib()
    ctxs = torch.randint(1, max_ctx + 1, (B,)).tolist()
    ctxs[0] = max_ctx
    max_pages = (max_ctx + 63) // 64
    nslots = B if not prefill else 4
    num_pages = nslots * max_pages
    kc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    vc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    perm = torch.randperm(num_pages).view(nslots, max_pages).int()
    if prefill:  # rows = (slot, position) pairs; several rows per slot
        row_slot = torch.randint(0, nslots, (B,), dtype=torch.int32)
        row_slot[5] = -1  # a padding row
        row_pos = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32)
        pos = torch.zeros(nslots, dtype=torch.int32)
    else:
        row_slot = torch.arange(B, dtype=torch.int32)
        row_pos = None
        pos = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32)
    q = torch.randn(B, nq, D, device="cuda").bfloat16()
    ws = lib.tps_attn_workspace(B, nq, D, 0)
    pm, po = torch.empty(ws // D, device="cuda"), torch.empty(ws, device="cuda")
    pl = torch.empty_like(pm)
    ctr = torch.zeros(B * nkv, dtype=torch.int32, device="cuda")
    out = torch.full((B, nq, D), 3.0, device="cuda", dtype=torch.bfloat16)
    rs_d, pos_d, pt_d = row_slot.cuda(), pos.cuda(), perm.cuda()
    rp_d = row_pos.cuda() if prefill else None
    for _ in range(2):  # second launch checks the merge counters re-armed
        nat.check(lib.tps_paged_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), rs_d.data_ptr(), pos_d.data_ptr(),
                                          rp_d.data_ptr() if prefill else None, pt_d.data_ptr(), max_pages, B, nq,
                                          nkv, D, 0, pm.data_ptr(), pl.data_ptr(), po.data_ptr(), ctr.data_ptr(),
                                          out.data_ptr(), None, 0, 0, None, None, None, _stream()))
        torch.cuda.synchronize()
        assert int(ctr.sum()) == 0
    valid = [b for b in range(B) if int(row_slot[b]) >= 0]
    tables = [perm[int(row_slot[b])].tolist() for b in valid]
    ref = _ref_attention(q.cpu()[valid], kc.cpu(), vc.cpu(), tables, [ctxs[b] - 1 for b in valid], nq // nkv)
    err = (out.float().cpu()[valid] - ref).abs().max().item()
    assert err < 2e-2, err
    if prefill:
        assert (out[5] == 0).all()


@pytest.mark.parametrize("mode", [0, 1])
def test_copy_items_bit_exact(mode):
    torch.manual_seed(mode)
    src = torch.randint(0, 256, (3 << 20,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    # ragged items: 16 B multiples, a large 1 MiB one, and an odd-size tail (LSU only)
    spec = [(0, 4096, 16384), (1600000, 1 << 20, 65536 - 16), (2 << 20, 1200000, 1 << 20)]
    if mode == 0:
        spec.append((12345, 2900000, 77))  # unaligned odd-size item: LSU byte tail
    items = torch.zeros((len(spec), 4), dtype=torch.int64)
    for i, (so, do, nb) in enumerate(spec):
        items[i, 0] = src.data_ptr() + so
        items[i, 1] = dst.data_ptr() + do
        items[i, 2] = nb
    items = items.cuda()
    nat.check(nat.lib().tps_copy_items(items.data_ptr(), len(spec), mode, 0, _stream()))
    torch.cuda.synchronize()
    want = torch.zeros_like(src)
    for so, do, nb in spec:
        want[do:do + nb] = src[so:so + nb]
    assert torch.equal(dst, want)


def test_barrier_epoch_slots_virtual():
    """Rank 0 of 4: stores the epoch into its slot of the three peers' arrays and waits on the
    three peer slots of its own array (pre-armed here as if the peers had arrived)."""
    mine = torch.zeros(4, dtype=torch.int64, device="cuda")
    peer_arrays = torch.zeros((3, 4), dtype=torch.int64, device="cuda")
    peers = nat.ptr_array([peer_arrays[i].data_ptr() for i in range(3)])  # slot 0 = this rank's
    for epoch in (1, 2, 5):
        mine[1:] = epoch
        nat.check(nat.lib().tps_barrier(peers, 3, mine.data_ptr(), 4, 0, epoch, _stream()))
        torch.cuda.synchronize()
        assert peer_arrays[:, 0].tolist() == [epoch] * 3 and peer_arrays[:, 1:].sum() == 0


@pytest.mark.parametrize("F,k,b", [(1024, 256, 1), (2368, 3584, 16), (18944, 3584, 64), (512, 512, 300)])
def test_linear_silu_fused_epilogue(F, k, b):
    """Gate/up GEMM with SwiGLU in the epilogue vs torch fp32 on the interleaved weight layout."""
    torch.manual_seed(F + b)
    w = (torch.randn(2 * F, k, device="cuda") * 0.05).bfloat16()   # rows: 64-blocks [gate c | up c]
    x = torch.randn(b, k, device="cuda").bfloat16()
    act = torch.zeros(b, F, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().tps_linear_silu(w.data_ptr(), 2 * F, k, k, x.data_ptr(), b, b, k, act.data_ptr(), F,
                                        _stream()))
    torch.cuda.synchronize()
    y = x.float() @ w.float().T                                       # [b, 2F]
    blk = y.view(b, F // 64, 2, 64)
    g, u = blk[:, :, 0, :].reshape(b, F), blk[:, :, 1, :].reshape(b, F)
    ref = torch.nn.functional.silu(g) * u
    err = (act.float() - ref).abs() / (ref.abs() + 1.0)
    assert err.max().item() < 2e-2


@pytest.mark.parametrize("n,k,b,ndst,splits", [(3584, 512, 1, 8, 2), (256, 128, 7, 2, 2), (3584, 2368, 64, 4, 4),
                                                 (3584, 512, 16, 8, 1)])
def test_linear_push_fused_allreduce_epilogue(n, k, b, ndst, splits):
    """tps_linear_push: every split partial lands in every destination (the peers' receive
    slots) at split * split_stride + row * n, rows >= b untouched, and the last CTA bumps
    every counter exactly once per launch (repeated launches / graph replays re-arm)."""
    torch.manual_seed(n + b)
    w = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    x = torch.randn(b, k, device="cuda").bfloat16()
    rows = 64
    slots = [torch.full((splits, rows, n), float("nan"), device="cuda") for _ in range(ndst)]
    ctrs = [torch.zeros(4, dtype=torch.int64, device="cuda") for _ in range(ndst)]
    done = torch.zeros(4, dtype=torch.int32, device="cuda")
    lib = nat.lib()
    for rep in range(3):
        nat.check(lib.tps_linear_push(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k,
                                      nat.ptr_array([t.data_ptr() for t in slots]), ndst, rows * n, splits,
                                      nat.ptr_array([c.data_ptr() + 8 for c in ctrs]), ndst,
                                      done.data_ptr() + 4, _stream()))
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    tol = 2e-3 * math.sqrt(k) * 0.05 * 4 + 1e-4
    for t, c in zip(slots, ctrs):
        got = t[:, :b].sum(0)
        assert (got - ref).abs().max().item() <= tol
        assert torch.equal(t[:, :b], slots[0][:, :b])
        assert torch.isnan(t[:, b:]).all()
        assert c.tolist() == [0, 3, 0, 0]
    assert done.tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("b,tp,splits", [(1, 8, 2), (5, 2, 4), (64, 4, 3)])
def test_ll_push_and_norm(b, tp, splits):
    """LL fused allreduce: tp 'ranks' push {value, tag} partials of their row-parallel
    projection into one receive area; tps_add_norm_ll polls the tags, sums the tp x splits
    slots in (rank, split) order, adds the residual and RMS-normalises."""
    from paper_2605_23945_b200.executor import FUSE_ROWS, FUSE_SOURCES
    torch.manual_seed(b * tp)
    H, K = 512, 256
    lib = nat.lib()
    ll = torch.zeros((FUSE_SOURCES, FUSE_ROWS, H), dtype=torch.int64, device="cuda")
    epoch = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    mult, phase = 11, 3
    ws = [(torch.randn(H, K, device="cuda") * 0.05).bfloat16() for _ in range(tp)]
    xs = [torch.randn(b, K, device="cuda").bfloat16() for _ in range(tp)]
    row = FUSE_ROWS * H * 8
    for r in range(tp):
        dst = ll.data_ptr() + r * splits * row
        nat.check(lib.tps_linear_push_ll(ws[r].data_ptr(), H, K, K, xs[r].data_ptr(), b, b, K,
                                         nat.ptr_array([dst]), 1, FUSE_ROWS * H, splits, epoch.data_ptr(), mult,
                                         phase, _stream()))
    torch.cuda.synchronize()
    tags = (ll[:tp * splits, :b] >> 32)
    assert (tags == 7 * mult + phase).all()
    resid = torch.randn(b, H, device="cuda")
    ref_resid = resid + sum(xs[r].float() @ ws[r].float().T for r in range(tp))
    wn = (torch.rand(H, device="cuda") + 0.5).bfloat16()
    out = torch.zeros(b, H, dtype=torch.bfloat16, device="cuda")
    ctr = torch.full((1,), 5, dtype=torch.int64, device="cuda")
    nat.check(lib.tps_add_norm_ll(resid.data_ptr(), ll.data_ptr(), tp * splits, FUSE_ROWS * H, epoch.data_ptr(),
                                  mult, phase, wn.data_ptr(), ctypes.c_float(1e-6), H, b, out.data_ptr(), H,
                                  ctr.data_ptr(), tp, _stream()))
    torch.cuda.synchronize()
    ref = ref_resid * torch.rsqrt(ref_resid.pow(2).mean(-1, keepdim=True) + 1e-6) * wn.float()
    assert (resid - ref_resid).abs().max().item() < 2e-3
    assert (out.float() - ref).abs().max().item() < 3e-2
    assert ctr.item() == 5 + tp  # the phase counter advanced as if the counter protocol had run



@pytest.mark.parametrize("D,nq,nkv,nslots,per,ragged", [(128, 28, 4, 8, 8, False), (128, 7, 1, 5, 20, True),
                                                         (128, 32, 8, 6, 16, True), (64, 4, 4, 9, 3, False),
                                                         (128, 16, 1, 3, 9, True)])
def test_grouped_prefill_attention(D, nq, nkv, nslots, per, ragged):
    """tps_prefill_attention (one CTA per sample group and KV head, per-row causal limits) vs
    torch fp32, on a position-major chunk with padding rows; groups cut at the executor's
    positions-per-group limit; rows outside every group stay untouched."""
    from paper_2605_23945_b200.executor import prefill_groups
    torch.manual_seed(D + nq + nslots)
    lib = nat.lib()
    G = nq // nkv
    gp = lib.tps_prefill_group_positions(G)
    assert gp == min(16, 64 // G)
    base = torch.randint(0, 900, (nslots,)).tolist()
    n_i = [per - (i % 3 if ragged else 0) for i in range(nslots)]
    rows_s, rows_p = [], []
    for j in range(per):
        for s in range(nslots):
            if j < n_i[s]:
                rows_s.append(s)
                rows_p.append(base[s] + j)
    R = len(rows_s) + 5
    rs = torch.tensor(rows_s + [-1] * 5, dtype=torch.int32)
    rp = torch.tensor(rows_p + [0] * 5, dtype=torch.int32)
    max_pages = (max(base) + per + 63) // 64 + 1
    num_pages = nslots * max_pages
    kc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    vc = torch.randn(num_pages, nkv, 64, D, device="cuda").bfloat16()
    perm = torch.randperm(num_pages).view(nslots, max_pages).int()
    q = torch.randn(R, nq, D, device="cuda").bfloat16()
    rows, n = prefill_groups(rs.numpy(), gp)
    assert int(n.sum()) == len(rows_s) and int((n > 0).sum()) >= nslots
    out = torch.full((R, nq, D), 5.0, device="cuda", dtype=torch.bfloat16)
    gr, gn = torch.from_numpy(rows).cuda(), torch.from_numpy(n).cuda()
    rs_d, rp_d, pt_d = rs.cuda(), rp.cuda(), perm.cuda()  # (kept alive across the launch)
    nat.check(lib.tps_prefill_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), rs_d.data_ptr(),
                                        rp_d.data_ptr(), gr.data_ptr(), gn.data_ptr(), R,
                                        pt_d.data_ptr(), max_pages, nq, nkv, D, out.data_ptr(), _stream()))
    torch.cuda.synchronize()
    valid = list(range(len(rows_s)))
    ref = _ref_attention(q.cpu()[valid], kc.cpu(), vc.cpu(), [perm[rows_s[b]].tolist() for b in valid],
                         [rows_p[b] for b in valid], G)
    err = (out.float().cpu()[valid] - ref).abs().max().item()
    assert err < 2e-2, err
    assert (out[len(rows_s):] == 5.0).all()


@pytest.mark.parametrize("n,k,b,ndst", [(3584, 2368, 1, 8), (3584, 512, 16, 8), (256, 128, 7, 2), (3584, 4736, 64, 4),
                                        (4096, 1792, 33, 8)])
def test_linear_push_ll_cluster(n, k, b, ndst):
    """tps_linear_push_ll_cluster: the split partials summed over DSMEM in split order equal
    tps_linear (same split count) + an in-order sum, bit for bit, in every destination as
    {value, tag}; rows >= b untouched."""
    lib = nat.lib()
    S = lib.tps_cluster_splits(n, k, b)
    assert S >= 1
    torch.manual_seed(n + k + b)
    w = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    x = torch.randn(b, k, device="cuda").bfloat16()
    ws = torch.zeros(S, b, n, device="cuda")
    nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k, ws.data_ptr(), S, _stream()))
    ref = torch.zeros(b, n, device="cuda")
    for s in range(S):
        ref += ws[s]
    epoch = torch.tensor([5], dtype=torch.int64, device="cuda")
    slots = [torch.full((b + 2, n), -1, dtype=torch.int64, device="cuda") for _ in range(ndst)]
    nat.check(lib.tps_linear_push_ll_cluster(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k,
                                             nat.ptr_array([t.data_ptr() for t in slots]), ndst, epoch.data_ptr(),
                                             3, 1, _stream()))
    torch.cuda.synchronize()
    # directly against torch fp32 too (not only transitively through tps_linear)
    fp32 = (x.float() @ w.float().T).cpu()
    tol = 2e-3 * math.sqrt(k) * 0.05 * 4 + 1e-4
    for t in slots:
        u = t[:b].cpu()
        tags = (u >> 32) & 0xFFFFFFFF
        assert (tags == 5 * 3 + 1).all()
        vals = (u & 0xFFFFFFFF).to(torch.int32).view(torch.float32)
        assert torch.equal(vals, ref.cpu())
        assert (vals - fp32).abs().max().item() <= tol
        assert (t[b:] == -1).all()


@pytest.mark.parametrize("V,k,b", [(4096, 256, 2), (152064, 3584, 64), (151936, 3584, 1), (19008, 3584, 17)])
def test_linear_argmax_epilogue(V, k, b):
    """tps_linear_argmax: logits equal tps_linear's (split-K 1) bit for bit, and the per-tile
    candidates merged by tps_argmax_finalize pick the row's max logit with the smallest index
    on ties -- the token of tps_argmax_stage1 + finalize."""
    lib = nat.lib()
    torch.manual_seed(V + b)
    w = (torch.randn(V, k, device="cuda") * 0.05).bfloat16()
    x = torch.randn(b, k, device="cuda").bfloat16()
    x[0] = 0  # a row of exact ties (all logits 0): the smallest index must win
    ref = torch.zeros(1, b, V, device="cuda")
    nat.check(lib.tps_linear(w.data_ptr(), V, k, k, x.data_ptr(), b, b, k, ref.data_ptr(), 1, _stream()))
    tiles = -(-V // 128)
    logits = torch.full((b, V), float("nan"), device="cuda")
    cand = torch.zeros(b, tiles, 2, dtype=torch.int32, device="cuda")
    vocab0 = 1000
    nat.check(lib.tps_linear_argmax(w.data_ptr(), V, k, k, x.data_ptr(), b, b, k, logits.data_ptr(),
                                    cand.data_ptr(), vocab0, _stream()))
    torch.cuda.synchronize()
    assert torch.equal(logits, ref[0])
    tol = 2e-3 * math.sqrt(k) * 0.05 * 4 + 1e-4  # and directly against torch fp32
    assert (logits - x.float() @ w.float().T).abs().max().item() <= tol
    vals = cand[..., 0].view(torch.float32).cpu()
    idxs = cand[..., 1].cpu()
    lg = ref[0].cpu()
    for i in range(b):
        t = int(vals[i].argmax())
        m = lg[i].max()
        assert vals[i, t] == m
        first = int((lg[i] == m).nonzero()[0])
        assert int(idxs[i][vals[i] == m].min()) == vocab0 + first
