"""Paged KV pool and per-sample slot state of one rank (the Cache Manager's data).

Layout (bf16): pool[layer][k|v][page][kv_head][64 tokens][head_dim]. One
(layer, k|v, page, kv_head) slice is a contiguous page_size*head_dim*2-byte
chunk (16 KB at D=128): the decode attention streams it and the Switch
Executor migrates it as one copy item.

Pages for a sample are reserved for its maximum context (prompt + l_max) at
admission -- the reference's admission rule per_node*(prompt+l_max) <= budget
(tpshift/engine.py:142-147) -- so the decode loop never allocates and a CUDA
graph replay only needs the row -> slot vector.

Per-slot state (history of token ids, next position, prompt length, page
table) is what a migration moves besides the KV pages (north star item 3).
"""

from __future__ import annotations

import torch

from .errors import ScenarioError

PAGE = 64


class KVPool:
    def __init__(self, num_layers: int, n_kv_local: int, head_dim: int, num_pages: int,
                 device: torch.device | str):
        self.num_layers = num_layers
        self.n_kv = n_kv_local
        self.head_dim = head_dim
        self.num_pages = num_pages
        self.device = torch.device(device)
        self.buf = torch.zeros((num_layers, 2, num_pages, n_kv_local, PAGE, head_dim),
                               dtype=torch.bfloat16, device=self.device)
        self._free = list(range(num_pages - 1, -1, -1))

    @property
    def chunk_bytes(self) -> int:
        """Bytes of one (layer, k|v, page, kv_head) slice."""
        return PAGE * self.head_dim * 2

    def ptr(self, layer: int, kv: int, page: int = 0, head: int = 0) -> int:
        return self.buf[layer, kv, page, head].data_ptr()

    def layer_ptrs(self, layer: int) -> tuple[int, int]:
        return self.buf[layer, 0].data_ptr(), self.buf[layer, 1].data_ptr()

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def alloc(self, n: int) -> list[int]:
        if n > len(self._free):
            raise ScenarioError(f"KV pool exhausted: need {n} pages, {len(self._free)} free")
        return [self._free.pop() for _ in range(n)]

    def release(self, pages) -> None:
        self._free.extend(reversed(list(pages)))

    def reset(self) -> None:
        """Every page free again (a cached layout being reused)."""
        self._free = list(range(self.num_pages - 1, -1, -1))


def pages_for(tokens: int) -> int:
    return (tokens + PAGE - 1) // PAGE


class SlotTable:
    """Device-resident per-sample state of one rank, indexed by slot."""

    def __init__(self, num_slots: int, max_len: int, device: torch.device | str):
        self.num_slots = num_slots
        self.max_len = max_len
        self.max_pages = pages_for(max_len)
        self.device = torch.device(device)
        self.history = torch.zeros((num_slots, max_len), dtype=torch.int32, device=self.device)
        self.pos = torch.zeros(num_slots, dtype=torch.int32, device=self.device)
        self.page_table = torch.zeros((num_slots, self.max_pages), dtype=torch.int32, device=self.device)
        # non-greedy sampler key per slot (uint64 bits; the rest of the sampler state is the position)
        self.seed = torch.zeros(num_slots, dtype=torch.int64, device=self.device)
        self._free = list(range(num_slots - 1, -1, -1))
        self.pages: dict[int, list[int]] = {}
        self.sample_of: dict[int, int] = {}

    def alloc(self, sample_id: int) -> int:
        if not self._free:
            raise ScenarioError("no free sample slot on this rank")
        s = self._free.pop()
        self.sample_of[s] = sample_id
        return s

    def release(self, slot: int) -> None:
        self.sample_of.pop(slot, None)
        self.pages.pop(slot, None)
        self._free.append(slot)

    def reset(self) -> None:
        """Every slot free again (a cached layout being reused)."""
        self._free = list(range(self.num_slots - 1, -1, -1))
        self.pages = {}
        self.sample_of = {}
