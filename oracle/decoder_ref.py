"""CPU ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

Never imported by the product package; never the thing measured as the GPU path.

Restates, on the CPU with simulated tensor-parallel ranks, the decode step the
B200 engine executes. The reference (`tpshift`) has no decode arithmetic -- it
prices a step with oracle_decode_latency (tpshift/latency.py:111-133) -- and the
paper's numerics live in SGLang 0.4.8 / PyTorch 2.7.1, which are
not vendored. This oracle therefore restates standard Llama / Qwen2 decoder
math (RMSNorm, rotate-half RoPE, GQA SDPA, SwiGLU, optional QKV bias) and pins
it against Hugging Face transformers' Qwen2ForCausalLM run in fp32 on the same
weights (tests/golden/make_decode_golden.py -> tests/golden/decode_tiny.npz).
Parity for decode numerics is therefore "pinned to transformers", not to the
reference (which has none): see DESIGN.md.

Two modes:
  round_bf16=False  pure fp32 math (the mode pinned against transformers);
  round_bf16=True   rounds to bf16 exactly where the B200 engine stores bf16:
                    normalised activations, q, K/V cache entries, attention
                    output, SiLU*up activations. Partial sums of row-parallel
                    projections are added to the fp32 residual rank by rank in
                    rank order (the engine's allreduce order).

The TP partition is restated here independently of the product code:
canonical contiguous slices (tpshift/reshard.py:25-43) applied per KV-head
group, with KV-head replication and an uneven (first parts larger) query-head
split when tp > n_kv (hard part 2).
"""

from __future__ import annotations

import math

import numpy as np
import torch


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def partition(geo: dict, tp: int, r: int) -> dict:
    nq, nkv = geo["n_q"], geo["n_kv"]
    G = nq // nkv
    if nkv % tp == 0:
        per = nkv // tp
        kv = (r * per, (r + 1) * per)
        q = (kv[0] * G, kv[1] * G)
    else:
        assert tp % nkv == 0
        m = tp // nkv
        h, sub = divmod(r, m)
        sizes = [G // m + (1 if i < G % m else 0) for i in range(m)]
        a = h * G + sum(sizes[:sub])
        q = (a, a + sizes[sub])
        kv = (h, h + 1)
    fw = geo["ffn"] // tp
    vw = geo["vocab"] // tp
    return {"q": q, "kv": kv, "ffn": (r * fw, (r + 1) * fw), "vocab": (r * vw, (r + 1) * vw)}


def rope_tables(head_dim: int, theta: float, max_pos: int):
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return (torch.from_numpy(np.cos(ang).astype(np.float32)),
            torch.from_numpy(np.sin(ang).astype(np.float32)))


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    var = (x * x).mean(dim=-1, keepdim=True)
    return x * torch.rsqrt(var + eps) * w


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [..., D]; cos/sin [..., D/2] broadcastable."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


class OracleDecoder:
    """Greedy decoder with `tp` simulated ranks over full fp32 weights.

    weights: {(layer, family): fp32 tensor} with the engine's full-tensor layout
      w_qkv [(nq+2nkv)*D, H] rows = [q heads | k heads | v heads], b_qkv [(nq+2nkv)*D],
      w_o [H, nq*D], w_gu [2F, H] rows = [gate | up], w_d [H, F], ln1/ln2 [H];
      layer -1: embed [V, H], ln_f [H], lm_head [V, H].
    """

    def __init__(self, geo: dict, weights: dict, tp: int = 1, round_bf16: bool = True,
                 max_len: int = 4096, threads: int | None = None):
        self.geo = geo
        self.tp = tp
        self.rb = round_bf16
        self.W = weights
        self.L = geo["num_layers"]
        self.D = geo["head_dim"]
        self.H = geo["hidden"]
        self.eps = geo["rms_eps"]
        self.cos, self.sin = rope_tables(self.D, geo["rope_theta"], max_len + 1)
        self.max_len = max_len
        if threads:
            torch.set_num_threads(threads)
        self.parts = [partition(geo, tp, r) for r in range(tp)]
        self.shards = [self._slice(p) for p in self.parts]
        self.cache: dict = {}

    def _r(self, x):
        return bf16(x) if self.rb else x

    def _slice(self, p: dict) -> dict:
        g, D = self.geo, self.D
        nq, nkv = g["n_q"], g["n_kv"]
        q0, q1 = p["q"]
        k0, k1 = p["kv"]
        f0, f1 = p["ffn"]
        v0, v1 = p["vocab"]
        out = {}
        if self.tp == 1:  # the single rank owns every tensor whole: views, no copies
            for l in range(self.L):
                for fam in ("w_qkv", "w_o", "w_gu", "w_d"):
                    out[(l, fam)] = self.W[(l, fam)]
                out[(l, "b_qkv")] = self.W.get((l, "b_qkv"))
            out.update(lm_head=self.W[(-1, "lm_head")], nq=nq, nkv=nkv, F=g["ffn"])
            return out
        for l in range(self.L):
            wqkv = self.W[(l, "w_qkv")]
            rows = list(range(q0 * D, q1 * D)) + list(range((nq + k0) * D, (nq + k1) * D)) + \
                list(range((nq + nkv + k0) * D, (nq + nkv + k1) * D))
            idx = torch.tensor(rows)
            out[(l, "w_qkv")] = wqkv[idx]
            b = self.W.get((l, "b_qkv"))
            out[(l, "b_qkv")] = b[idx] if b is not None else None
            out[(l, "w_o")] = self.W[(l, "w_o")][:, q0 * D:q1 * D]
            gu = self.W[(l, "w_gu")]
            F = g["ffn"]
            out[(l, "w_gu")] = torch.cat([gu[f0:f1], gu[F + f0:F + f1]], dim=0)
            out[(l, "w_d")] = self.W[(l, "w_d")][:, f0:f1]
        out["lm_head"] = self.W[(-1, "lm_head")][v0:v1]
        out["nq"] = q1 - q0
        out["nkv"] = k1 - k0
        out["F"] = f1 - f0
        return out

    def _kv(self, sample: int, layer: int, rank: int):
        key = (sample, layer, rank)
        if key not in self.cache:
            nkv = self.shards[rank]["nkv"]
            self.cache[key] = (torch.zeros(self.max_len, nkv, self.D), torch.zeros(self.max_len, nkv, self.D))
        return self.cache[key]

    def seed_context(self, sample: int, k_full: torch.Tensor, v_full: torch.Tensor) -> None:
        """Install a synthetic context for positions [0, P): k_full / v_full [L, P, n_kv, D]
        (post-RoPE K and V of every KV head, bf16-representable) -- the state a prefill of P
        tokens would leave; each simulated rank keeps its own KV heads."""
        P = k_full.shape[1]
        for l in range(self.L):
            for r, p in enumerate(self.parts):
                k0, k1 = p["kv"]
                kc, vc = self._kv(sample, l, r)
                kc[:P] = k_full[l, :, k0:k1]
                vc[:P] = v_full[l, :, k0:k1]

    @torch.no_grad()
    def prefill(self, tokens, sample: int, start: int = 0) -> torch.Tensor:
        """Positions start .. start+T-1 of one sample in one pass (causal attention over
        the cached context plus the chunk), the same rounding points as step(); returns
        the fp32 logits of the last position [V]. Equivalent to T calls of step()."""
        g, D = self.geo, self.D
        T = len(tokens)
        pos = torch.arange(start, start + T)
        x = self.W[(-1, "embed")][torch.tensor(tokens)].clone()
        cos, sin = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        scale = 1.0 / math.sqrt(D)
        S = start + T
        causal = torch.arange(S)[None, :] > pos[:, None]  # [T, S] True = masked
        for l in range(self.L):
            xn = self._r(rms_norm(x, self.W[(l, "ln1")], self.eps))
            partials = []
            for r, sh in enumerate(self.shards):
                nq, nkv = sh["nq"], sh["nkv"]
                qkv = xn @ sh[(l, "w_qkv")].T
                if sh[(l, "b_qkv")] is not None:
                    qkv = qkv + sh[(l, "b_qkv")]
                q = self._r(rope(qkv[:, :nq * D].view(T, nq, D), cos, sin))
                k = self._r(rope(qkv[:, nq * D:(nq + nkv) * D].view(T, nkv, D), cos, sin))
                v = self._r(qkv[:, (nq + nkv) * D:].reshape(T, nkv, D))
                kc, vc = self._kv(sample, l, r)
                kc[start:S] = k
                vc[start:S] = v
                G = nq // nkv
                kk = kc[:S].repeat_interleave(G, dim=1)  # [S, nq, D]
                vv = vc[:S].repeat_interleave(G, dim=1)
                s = torch.einsum("thd,shd->hts", q, kk) * scale
                s = s.masked_fill(causal[None], float("-inf"))
                o = torch.einsum("hts,shd->thd", torch.softmax(s, dim=-1), vv)
                partials.append(self._r(o).reshape(T, nq * D) @ sh[(l, "w_o")].T)
            for p_ in partials:
                x = x + p_
            xn = self._r(rms_norm(x, self.W[(l, "ln2")], self.eps))
            partials = []
            for sh in self.shards:
                gu = xn @ sh[(l, "w_gu")].T
                F = sh["F"]
                act = self._r(torch.nn.functional.silu(gu[:, :F]) * gu[:, F:])
                partials.append(act @ sh[(l, "w_d")].T)
            for p_ in partials:
                x = x + p_
        xn = self._r(rms_norm(x[-1:], self.W[(-1, "ln_f")], self.eps))
        return torch.cat([xn @ sh["lm_head"].T for sh in self.shards], dim=1)[0]

    def _attend(self, q, k, v, positions, samples, l, r):
        """Decode attention of B rows against their cached contexts (rows' own K/V appended
        first). One batched masked SDPA over the padded contexts (vectorised over rows)."""
        B, nq, D = q.shape
        nkv = k.shape[1]
        G = nq // nkv
        for i in range(B):
            kc, vc = self._kv(samples[i], l, r)
            kc[positions[i]] = k[i]
            vc[positions[i]] = v[i]
        S = max(positions) + 1
        K = torch.stack([self._kv(s, l, r)[0][:S] for s in samples])  # [B, S, nkv, D]
        V = torch.stack([self._kv(s, l, r)[1][:S] for s in samples])
        qg = q.view(B, nkv, G, D)
        s = torch.einsum("bkgd,bskd->bkgs", qg, K) / math.sqrt(D)
        mask = torch.arange(S)[None, :] > torch.tensor(positions)[:, None]  # [B, S]
        s = s.masked_fill(mask[:, None, None, :], float("-inf"))
        o = torch.einsum("bkgs,bskd->bkgd", torch.softmax(s, dim=-1), V)
        return o.reshape(B, nq, D)

    @torch.no_grad()
    def step(self, tokens, positions, samples) -> torch.Tensor:
        """One decode round: row i processes token tokens[i] at position positions[i]
        of sample samples[i] (its K/V for earlier positions must already be cached).
        Returns fp32 logits [B, V] (vocab shards concatenated in rank order)."""
        g, D, H = self.geo, self.D, self.H
        B = len(tokens)
        pos = torch.tensor(positions)
        x = self.W[(-1, "embed")][torch.tensor(tokens)].clone()
        cos, sin = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        for l in range(self.L):
            xn = self._r(rms_norm(x, self.W[(l, "ln1")], self.eps))
            partials = []
            for r, sh in enumerate(self.shards):
                nq, nkv = sh["nq"], sh["nkv"]
                qkv = xn @ sh[(l, "w_qkv")].T
                if sh[(l, "b_qkv")] is not None:
                    qkv = qkv + sh[(l, "b_qkv")]
                q = qkv[:, :nq * D].view(B, nq, D)
                k = qkv[:, nq * D:(nq + nkv) * D].view(B, nkv, D)
                v = qkv[:, (nq + nkv) * D:].view(B, nkv, D)
                q = self._r(rope(q, cos, sin))
                k = self._r(rope(k, cos, sin))
                v = self._r(v)
                o = self._r(self._attend(q, k, v, positions, samples, l, r)).reshape(B, nq * D)
                partials.append(o @ sh[(l, "w_o")].T)
            for p_ in partials:
                x = x + p_
            xn = self._r(rms_norm(x, self.W[(l, "ln2")], self.eps))
            partials = []
            for sh in self.shards:
                gu = xn @ sh[(l, "w_gu")].T
                F = sh["F"]
                gt, up = gu[:, :F], gu[:, F:]
                act = self._r(torch.nn.functional.silu(gt) * up)
                partials.append(act @ sh[(l, "w_d")].T)
            for p_ in partials:
                x = x + p_
        xn = self._r(rms_norm(x, self.W[(-1, "ln_f")], self.eps))
        return torch.cat([xn @ sh["lm_head"].T for sh in self.shards], dim=1)


def greedy(logits: torch.Tensor) -> list[int]:
    """argmax with the smallest index on ties (the engine's tie rule)."""
    m = logits.max(dim=1, keepdim=True).values
    idx = torch.arange(logits.shape[1]).expand_as(logits)
    return torch.where(logits == m, idx, logits.shape[1]).min(dim=1).values.tolist()


def numpy_weights(geo: dict, seed: int) -> dict:
    """Deterministic bf16-representable fp32 weights from numpy's PCG64 (portable)."""
    rng = np.random.default_rng(seed)
    H, D, F, V = geo["hidden"], geo["head_dim"], geo["ffn"], geo["vocab"]
    nq, nkv = geo["n_q"], geo["n_kv"]

    def t(*shape, base=0.0):
        a = rng.standard_normal(shape).astype(np.float32) * 0.02 + base
        return bf16(torch.from_numpy(a))

    W = {(-1, "embed"): t(V, H), (-1, "ln_f"): t(H, base=1.0), (-1, "lm_head"): t(V, H)}
    for l in range(geo["num_layers"]):
        W[(l, "w_qkv")] = t((nq + 2 * nkv) * D, H)
        if geo.get("qkv_bias", True):
            W[(l, "b_qkv")] = t((nq + 2 * nkv) * D)
        W[(l, "w_o")] = t(H, nq * D)
        W[(l, "w_gu")] = t(2 * F, H)
        W[(l, "w_d")] = t(H, F)
        W[(l, "ln1")] = t(H, base=1.0)
        W[(l, "ln2")] = t(H, base=1.0)
    return W


TINY = dict(num_layers=2, hidden=256, n_q=4, n_kv=2, head_dim=64, ffn=1024, vocab=4096,
            qkv_bias=True, rope_theta=10000.0, rms_eps=1e-6)
