"""CPU ORACLE -- test infrastructure only: the engine's stochastic sampler, restated.

Counter-based sampling makes a sample's sampler state two integers -- its key (seed)
and the position being sampled -- so migrating a sample across TP layouts moves no RNG
state beyond its position (which the Switch Executor already moves) and its seed.
Token at position p+1 of a sample with key s and temperature T:

    argmax_v  logit_v / T + Gumbel(u_v),   u_v = philox4x32_10(ctr=(p+1, v, 0, 0), key=s).x

(Gumbel-max: an exact draw from softmax(logit / T)). The 32-bit Philox output is mapped
to u = ((x >> 8) + 0.5) / 2^24 and Gumbel(u) = -log(-log(u)), evaluated in float32 like
the kernel. Philox4x32-10 is Salmon et al., "Parallel random numbers: as easy as
1, 2, 3" (SC'11); tests/test_sampler_ref.py checks it against the Random123
known-answer vectors.
"""

from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """ctr: 4 uint32 arrays (broadcastable), key: 2 uint32 scalars/arrays -> 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) for c in ctr)
    k0, k1 = (np.asarray(k, dtype=np.uint64) for k in key)
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def gumbel(x: np.ndarray) -> np.ndarray:
    u = ((x >> np.uint32(8)).astype(np.float32) + np.float32(0.5)) * np.float32(1.0 / (1 << 24))
    return -np.log(-np.log(u, dtype=np.float32), dtype=np.float32)


def sample_scores(logits: np.ndarray, seed: int, pos_next: int, temperature: float) -> np.ndarray:
    """Perturbed scores logit / T + Gumbel of one row (vocab order)."""
    V = logits.shape[-1]
    v = np.arange(V, dtype=np.uint64)
    x, _, _, _ = philox4x32_10((np.uint64(pos_next), v, 0, 0), (seed & MASK, (seed >> 32) & MASK))
    return logits.astype(np.float32) * np.float32(1.0 / temperature) + gumbel(x)


def sample(logits: np.ndarray, seed: int, pos_next: int, temperature: float) -> int:
    s = sample_scores(logits, seed, pos_next, temperature)
    return int(np.argmax(s))  # smallest index on ties, like the kernel


def seed_of(run_seed: int, sample_id: int) -> int:
    """Per-sample key (the engine's `sampler_seed`): splitmix64 of (run seed, sample id)."""
    z = (run_seed * 0x9E3779B97F4A7C15 + sample_id + 1) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)
