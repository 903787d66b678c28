"""Random-init weights and their per-rank canonical shards, packed in one arena.

Weights are synthetic (no checkpoints offline): every full tensor is drawn from
its own seeded stream, so any rank can materialise exactly its shard without
communication and two layouts of the same model are bit-identical views of
the same logical weights -- which is what makes a reshard checkable byte for
byte. Linear weights and biases ~ N(0, 0.02) (HF initializer_range), norm
weights 1 + N(0, 0.02) (non-trivial so a mis-indexed norm is visible).

All of a rank's tensors live in one contiguous uint8 arena (256-byte aligned
slices): one IPC handle exposes the whole shard set to NVLink peers and the old
layout is released in one free after a switch.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import torch

from .models import (GLOBAL_FAMILIES, DecoderGeometry, RankShard, full_shape, layer_families,
                     shard_ranges, shard_shape)

_ALIGN = 256


def _stream_seed(seed: int, layer: int, family: str) -> int:
    h = hashlib.blake2b(f"{seed}/{layer}/{family}".encode(), digest_size=8).digest()
    return int.from_bytes(h, "little") & ((1 << 63) - 1)


def full_tensor(geom: DecoderGeometry, family: str, layer: int, seed: int,
                device: torch.device | str) -> torch.Tensor:
    """The full (unsharded) bf16 tensor ``family`` of ``layer`` (layer -1 = global)."""
    shape = full_shape(geom, family)
    gen = torch.Generator(device=device)
    gen.manual_seed(_stream_seed(seed, layer, family))
    t = torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
    t.mul_(0.02)
    if family in ("ln1", "ln2", "ln_f"):
        t.add_(1.0)
    return t.to(torch.bfloat16)


def slice_shard(geom: DecoderGeometry, family: str, full: torch.Tensor, sh: RankShard) -> torch.Tensor:
    axis, ranges = shard_ranges(geom, family, sh)
    parts = [full.narrow(axis, a, b - a) for a, b in ranges]
    return parts[0] if len(parts) == 1 else torch.cat(parts, dim=axis)


@dataclass
class ArenaLayout:
    """Byte offsets of every (layer, family) tensor of one rank's shard set."""

    entries: dict[tuple[int, str], tuple[int, tuple[int, ...]]]
    total_bytes: int


def arena_layout(geom: DecoderGeometry, sh: RankShard) -> ArenaLayout:
    entries = {}
    off = 0
    keys = [(-1, f) for f in GLOBAL_FAMILIES]
    keys += [(l, f) for l in range(geom.num_layers) for f in layer_families(geom)]
    for layer, fam in keys:
        shape = shard_shape(geom, fam, sh)
        nbytes = 2
        for d in shape:
            nbytes *= d
        entries[(layer, fam)] = (off, shape)
        off += (nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
    return ArenaLayout(entries=entries, total_bytes=off)


class RankWeights:
    """One TP rank's shard set: a single device arena plus bf16 views into it."""

    def __init__(self, geom: DecoderGeometry, shard: RankShard, device: torch.device | str,
                 arena: torch.Tensor | None = None):
        self.geom = geom
        self.shard = shard
        self.device = torch.device(device)
        self.layout = arena_layout(geom, shard)
        if arena is None:
            arena = torch.empty(self.layout.total_bytes, dtype=torch.uint8, device=self.device)
        assert arena.numel() >= self.layout.total_bytes
        self.arena = arena
        self.views: dict[tuple[int, str], torch.Tensor] = {}
        for key, (off, shape) in self.layout.entries.items():
            n = 1
            for d in shape:
                n *= d
            self.views[key] = arena[off:off + 2 * n].view(torch.bfloat16).view(shape)

    def __getitem__(self, key: tuple[int, str]) -> torch.Tensor:
        return self.views[key]

    def tensor_ptr(self, layer: int, family: str) -> int:
        return self.views[(layer, family)].data_ptr()

    @property
    def nbytes(self) -> int:
        return self.layout.total_bytes

    def fill_random(self, seed: int) -> "RankWeights":
        """Materialise this rank's shards from the seeded full tensors (on this device)."""
        for (layer, fam), view in self.views.items():
            full = full_tensor(self.geom, fam, layer, seed, self.device)
            view.copy_(slice_shard(self.geom, fam, full, self.shard))
            del full
        return self

    @classmethod
    def random(cls, geom: DecoderGeometry, shard: RankShard, device, seed: int) -> "RankWeights":
        return cls(geom, shard, device).fill_random(seed)
