"""The tail-batch warp-shuffle GEMV (csrc/gemv.cu, VERDICT row N1) on a B200.

Kernel level: tps_gemv / tps_gemv_silu / tps_gemv_push_ll / tps_gemv_argmax against a torch
float64 matmul of the same bf16 operands, at the true Qwen2.5-7B projection shapes of TP1 and
TP8 shards plus ragged ones, b = 1..4. Tolerance (stated): fp32 accumulation of bf16 products,
|d| <= 2e-3 * sqrt(K) * 0.05 * 4 + 1e-4 (the tcgen05 projection tests' bound); SwiGLU
activations are bf16, so within one bf16 ulp (2^-7 relative) of the float64 SwiGLU; the LL
push and the argmax logits equal tps_gemv's outputs bit for bit (same reduction), and the
greedy candidates pick each tile's max with the smallest index on ties. Rows >= b of the
activations hold NaN and must never be read; output rows >= b must stay untouched.

Step level: decode with every projection on the GEMV (executor.gemv_rows = 4) against the
CPU oracle at the tolerance of tests/test_gpu_decode.py (|dlogit| <= 0.05, greedy tokens
equal where the oracle's top-2 margin > 0.1), mini geometries at TP1/2/4/8 and the true
c2/c3/c4 per-layer shapes at 8K/16K contexts.
"""

import math

import pytest
import torch

from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.errors import ConfigError

pytestmark = pytest.mark.gpu

SHAPES = [
    (576, 3584), (3584, 448), (4736, 3584), (3584, 2368),      # Qwen2.5-7B TP8 shard: QKV, O, gate/up, down
    (4608, 3584), (3584, 3584), (37888, 3584), (3584, 18944),  # TP1
    (1000, 104), (5, 8), (130, 520), (19008, 3584)]            # ragged / LM-head shard


@pytest.fixture(scope="module", autouse=True)
def _init():
    nat.init_device(0)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _operands(n, k, b, seed):
    torch.manual_seed(seed)
    w = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    x = torch.full((b + 2, k), float("nan"), device="cuda").bfloat16()  # rows >= b are never read
    x[:b] = torch.randn(b, k, device="cuda").bfloat16()
    return w, x


def _tol(k):
    return 2e-3 * math.sqrt(k) * 0.05 * 4 + 1e-4


def test_gemv_max_rows():
    assert nat.lib().tps_gemv_max_rows() == 4


@pytest.mark.parametrize("n,k", SHAPES)
@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_gemv_matches_fp64(n, k, b):
    lib = nat.lib()
    w, x = _operands(n, k, b, n + k + b)
    ref = x[:b].double() @ w.double().T
    out = torch.full((b + 1, n), -7.0, device="cuda")
    nat.check(lib.tps_gemv(w.data_ptr(), n, k, k, x.data_ptr(), b, k, out.data_ptr(), _stream()))
    torch.cuda.synchronize()
    assert torch.isfinite(out[:b]).all()
    assert (out[:b].double() - ref).abs().max().item() <= _tol(k)
    assert (out[b:] == -7.0).all()


@pytest.mark.parametrize("n,k", [(4736, 3584), (37888, 3584), (256, 256), (128, 64), (3584, 2368)])
@pytest.mark.parametrize("b", [1, 3, 4])
def test_gemv_silu_matches_fp64(n, k, b):
    """W rows in 64-row [gate c | up c] blocks (the weight arena's layout); act = bf16(silu(g) * u)."""
    lib = nat.lib()
    w, x = _operands(n, k, b, 7 * n + k + b)
    F = n // 2
    y = x[:b].double() @ w.double().T  # [b, n]
    blk = y.view(b, n // 128, 2, 64)
    g, u = blk[:, :, 0].reshape(b, F), blk[:, :, 1].reshape(b, F)
    ref = g / (1 + torch.exp(-g)) * u
    act = torch.full((b + 1, F + 8), -3.0, device="cuda").bfloat16()
    nat.check(lib.tps_gemv_silu(w.data_ptr(), n, k, k, x.data_ptr(), b, k, act.data_ptr(), F + 8, _stream()))
    torch.cuda.synchronize()
    got = act[:b, :F].double()
    err = (got - ref).abs()
    assert (err <= ref.abs() * 2.0 ** -7 + _tol(k) * (1 + ref.abs())).all(), err.max().item()
    assert (act[b:] == -3.0).all() and (act[:b, F:] == -3.0).all()


@pytest.mark.parametrize("n,k,b,ndst", [(3584, 448, 1, 8), (3584, 2368, 4, 8), (3584, 18944, 2, 1),
                                        (4096, 1792, 3, 4), (200, 64, 4, 2)])
def test_gemv_push_ll(n, k, b, ndst):
    """One LL {fp32 bits, tag} per element in every destination at dst + i * n + j, the value
    equal to tps_gemv's bit for bit; rows >= b untouched."""
    lib = nat.lib()
    w, x = _operands(n, k, b, n * 3 + k + b)
    ref = torch.zeros(b, n, device="cuda")
    nat.check(lib.tps_gemv(w.data_ptr(), n, k, k, x.data_ptr(), b, k, ref.data_ptr(), _stream()))
    epoch = torch.tensor([9], dtype=torch.int64, device="cuda")
    slots = [torch.full((b + 2, n), -1, dtype=torch.int64, device="cuda") for _ in range(ndst)]
    nat.check(lib.tps_gemv_push_ll(w.data_ptr(), n, k, k, x.data_ptr(), b, k,
                                   nat.ptr_array([t.data_ptr() for t in slots]), ndst, epoch.data_ptr(), 5, 2,
                                   _stream()))
    torch.cuda.synchronize()
    for t in slots:
        u = t[:b].cpu()
        assert (((u >> 32) & 0xFFFFFFFF) == 9 * 5 + 2).all()
        vals = (u & 0xFFFFFFFF).to(torch.int32).view(torch.float32)
        assert torch.equal(vals, ref.cpu())
        assert (t[b:] == -1).all()


@pytest.mark.parametrize("V,k,b", [(4096, 256, 2), (152064, 3584, 1), (19008, 3584, 4), (1000, 64, 3)])
def test_gemv_argmax(V, k, b):
    """Logits equal tps_gemv's bit for bit; per (row, 128-column tile) the candidate is the tile's
    max logit with the smallest vocab index on ties (tps_linear_argmax's contract)."""
    lib = nat.lib()
    w, x = _operands(V, k, b, V + b)
    x[0] = 0  # a row of exact ties (every logit 0): the smallest index must win
    ref = torch.zeros(b, V, device="cuda")
    nat.check(lib.tps_gemv(w.data_ptr(), V, k, k, x.data_ptr(), b, k, ref.data_ptr(), _stream()))
    tiles = -(-V // 128)
    logits = torch.full((b, V), float("nan"), device="cuda")
    cand = torch.zeros(b, tiles, 2, dtype=torch.int32, device="cuda")
    vocab0 = 500
    nat.check(lib.tps_gemv_argmax(w.data_ptr(), V, k, k, x.data_ptr(), b, k, logits.data_ptr(), cand.data_ptr(),
                                  vocab0, _stream()))
    torch.cuda.synchronize()
    assert torch.equal(logits, ref)
    vals = cand[..., 0].view(torch.float32).cpu()
    idxs = cand[..., 1].cpu()
    lg = ref.cpu()
    for i in range(b):
        for t in range(tiles):
            seg = lg[i, 128 * t:128 * (t + 1)]
            m = seg.max()
            assert vals[i, t] == m
            assert idxs[i, t] == vocab0 + 128 * t + int((seg == m).nonzero()[0])


def test_gemv_rejects_bad_args():
    lib = nat.lib()
    w = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(8, 128, device="cuda")
    with pytest.raises(ConfigError):  # more rows than the GEMV form takes
        nat.check(lib.tps_gemv(w.data_ptr(), 128, 64, 64, w.data_ptr(), 5, 64, out.data_ptr(), _stream()))
    with pytest.raises(ConfigError):  # K not a multiple of 8
        nat.check(lib.tps_gemv(w.data_ptr(), 128, 60, 64, w.data_ptr(), 1, 64, out.data_ptr(), _stream()))
    with pytest.raises(ConfigError):  # SwiGLU needs n = 2F, F % 64 == 0
        nat.check(lib.tps_gemv_silu(w.data_ptr(), 96, 64, 64, w.data_ptr(), 1, 64, out.data_ptr(), 48, _stream()))


@pytest.fixture
def gemv_on(monkeypatch):
    from paper_2605_23945_b200 import executor
    monkeypatch.setattr(executor, "GEMV_ROWS", 4)


PROMPTS = [[5, 17, 300, 9, 4000, 1, 2, 3], [42, 42, 42, 7, 7, 7, 1000, 2047]]


@pytest.mark.parametrize("name,tp", [("tiny", 1), ("tiny", 2), ("mini-qwen", 4), ("mini-llama", 8),
                                     ("mini-qwen32", 2)])
def test_decode_on_gemv_matches_oracle(gemv_on, name, tp):
    from test_gpu_decode import run_parity
    run_parity(name, tp, PROMPTS, gen=8)


@pytest.mark.parametrize("name,tp,ctx", [("qwen2.5-7b", 1, [8190, 5000, 777, 64]),
                                         ("qwen2.5-7b", 8, [8190, 5000, 777, 64]),
                                         ("llama3-8b", 8, [16380, 9000, 130]),
                                         ("qwen2.5-32b", 8, [16380, 64])])
def test_full_shapes_on_gemv_match_oracle(name, tp, ctx):
    from test_gpu_decode_fullshape import run_long_context
    run_long_context(name, tp, ctx=ctx, gemv=4)


@pytest.mark.parametrize("name,tp", [("tiny", 2), ("mini-llama", 8)])
def test_gemv_graph_replay_matches_eager(gemv_on, name, tp):
    """The GEMV launches captured in a CUDA graph (as the bench and the stages run them) give the
    eager step's tokens bit for bit."""
    from paper_2605_23945_b200.group import admit, build_group
    from paper_2605_23945_b200.models import geometry
    geom = geometry(name)
    outs = []
    for graphs in (False, True):
        ranks, runner = build_group(geom, tp, max_batch=8, num_slots=4, max_len=128, seed=3, use_graphs=graphs)
        assert all(r.executor.gemv_rows == 4 for r in ranks)
        slots = [admit(ranks, i, p, max_ctx=len(p) + 20) for i, p in enumerate(PROMPTS)]
        runner.set_rows(2, slots)
        runner.step(2, 1)  # eager warm-up step
        if graphs:
            runner.capture(2)
        runner.step(2, 20)
        torch.cuda.synchronize()
        outs.append(ranks[0].slots.history[slots].cpu())
    assert torch.equal(outs[0], outs[1])
