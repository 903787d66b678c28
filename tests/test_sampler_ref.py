"""Philox4x32-10 of the sampler oracle against the Random123 known-answer vectors."""

import numpy as np

from oracle.sampler_ref import philox4x32_10, sample, seed_of

KAT = [  # (ctr[4], key[2]) -> out[4]   (Random123 kat_vectors, philox4x32 R=10)
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_known_answers():
    for ctr, key, want in KAT:
        got = philox4x32_10(ctr, key)
        assert tuple(int(x) for x in got) == want


def test_gumbel_max_draws_follow_softmax():
    logits = np.array([2.0, 1.0, 0.0, -1.0], dtype=np.float32)
    p = np.exp(logits) / np.exp(logits).sum()
    n = 20000
    counts = np.bincount([sample(logits, seed_of(7, i), 10, 1.0) for i in range(n)], minlength=4) / n
    assert np.abs(counts - p).max() < 0.015
    # temperature -> 0 approaches greedy
    assert sample(logits, seed_of(1, 2), 3, 1e-4) == 0


def test_product_sampler_key_matches_oracle():
    from paper_2605_23945_b200.workload import as_int64, sampler_seed
    for r in (0, 4, 123456789):
        for i in (0, 1, 511, 10**6):
            assert sampler_seed(r, i) == seed_of(r, i)
            k = as_int64(sampler_seed(r, i))
            assert -(1 << 63) <= k < (1 << 63) and (k & ((1 << 64) - 1)) == seed_of(r, i)
