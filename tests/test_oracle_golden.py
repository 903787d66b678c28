"""Pins the decode oracle (oracle/decoder_ref.py) before any GPU test trusts it.

tests/golden/decode_tiny.npz holds Hugging Face transformers' Qwen2ForCausalLM logits
(fp32, eager attention) for the tiny geometry on the oracle's numpy weights
(generator: tests/golden/make_decode_golden.py). The reference (tpshift) has no
decode numerics (it prices steps with tpshift/latency.py:111-133), so the decode
oracle is pinned to this independent implementation of the same decoder math.
"""

import os

import numpy as np
import pytest
import torch

from oracle.decoder_ref import TINY, OracleDecoder, numpy_weights

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decode_tiny.npz")
PIN_TOL = 1e-5  # fp32 vs fp32: only summation order differs


@pytest.fixture(scope="module")
def golden():
    z = np.load(GOLDEN)
    return z["logits"], z["prompts"].tolist(), int(z["seed"])


@pytest.mark.parametrize("tp", [1, 2])
def test_oracle_step_matches_transformers(golden, tp):
    logits, prompts, seed = golden
    orc = OracleDecoder(TINY, numpy_weights(TINY, seed), tp=tp, round_bf16=False, max_len=64)
    B, T = len(prompts), len(prompts[0])
    worst = 0.0
    for t in range(T):
        out = orc.step([p[t] for p in prompts], [t] * B, list(range(B))).numpy()
        worst = max(worst, float(np.abs(out - logits[:, t]).max()))
    assert worst <= PIN_TOL, worst


@pytest.mark.parametrize("tp", [1, 2])
def test_oracle_prefill_matches_transformers(golden, tp):
    """The batched causal prefill form, in two chunks, equals the golden last-position logits."""
    logits, prompts, seed = golden
    orc = OracleDecoder(TINY, numpy_weights(TINY, seed), tp=tp, round_bf16=False, max_len=64)
    for b, p in enumerate(prompts):
        orc.prefill(p[:5], b)
        out = orc.prefill(p[5:], b, start=5).numpy()
        assert float(np.abs(out - logits[b, -1]).max()) <= PIN_TOL


def test_oracle_prefill_equals_steps_bf16():
    """bf16-rounding mode: prefill of a chunk == the same positions decoded one by one."""
    W = numpy_weights(TINY, 7)
    prompt = [3, 1, 4, 1, 5, 9, 2, 6, 5, 3]
    a = OracleDecoder(TINY, W, tp=2, round_bf16=True, max_len=32)
    b = OracleDecoder(TINY, W, tp=2, round_bf16=True, max_len=32)
    last = a.prefill(prompt, 0)
    for t, tok in enumerate(prompt):
        ref = b.step([tok], [t], [0])[0]
    # bf16-rounded intermediates: the chunk's GEMMs and the per-position steps sum in a different
    # order (and the BLAS kernel the host picks changes that order again), so an intermediate can
    # land one bf16 ulp (2^-8 relative) apart; measured 1.4e-3 on logits of magnitude ~1.
    assert float((last - ref).abs().max()) <= 1e-2
    for l in range(TINY["num_layers"]):
        for r in range(2):
            ka, va = a._kv(0, l, r)
            kb, vb = b._kv(0, l, r)
            assert torch.allclose(ka, kb, atol=1e-2) and torch.allclose(va, vb, atol=1e-2)


def test_oracle_seeded_context_equals_cache_state():
    """seed_context installs exactly the per-rank KV-head slices a prefill would leave."""
    W = numpy_weights(TINY, 3)
    a = OracleDecoder(TINY, W, tp=2, round_bf16=True, max_len=32)
    a.prefill([7, 8, 9, 10], 0)
    L, P, nkv, D = TINY["num_layers"], 4, TINY["n_kv"], TINY["head_dim"]
    k = torch.zeros(L, P, nkv, D)
    v = torch.zeros(L, P, nkv, D)
    for l in range(L):
        for r, part in enumerate(a.parts):
            k0, k1 = part["kv"]
            k[l, :, k0:k1] = a._kv(0, l, r)[0][:P]
            v[l, :, k0:k1] = a._kv(0, l, r)[1][:P]
    b = OracleDecoder(TINY, W, tp=2, round_bf16=True, max_len=32)
    b.seed_context(0, k, v)
    assert torch.equal(a.step([11], [4], [0]), b.step([11], [4], [0]))
