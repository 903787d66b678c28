"""CPU ORACLE -- test infrastructure only (tests/, smoke(), bench cpu_baseline); never product code.

Restates the Switch Executor's data-movement semantics on the CPU:

* canonical target shards (tpshift/reshard.py:25-43 ShardLayout.rank_slice,
  applied per tensor family with the GQA head rule of decoder_ref.partition):
  the bytes every target rank must hold after a weight reshard;
* merge-first KV migration (tpshift/reshard.py:113-151): after the switch a
  sample's K/V for kv head h, layer l, token t equals its value before the
  switch, whichever rank held it;
* a byte-addressed memory simulator that executes copy items
  (src_ptr, dst_ptr, bytes) exactly like tps_copy_items, so a plan can be
  executed on the CPU and its result compared byte-for-byte.
"""

from __future__ import annotations

import numpy as np
import torch

from .decoder_ref import partition


def expected_shard(geo: dict, full: dict, tp: int, rank: int, layer: int, family: str) -> torch.Tensor:
    """The canonical shard of one tensor (bf16) for TP rank `rank` of `tp`."""
    p = partition(geo, tp, rank)
    D, nq, nkv, F = geo["head_dim"], geo["n_q"], geo["n_kv"], geo["ffn"]
    t = full[(layer, family)]
    q0, q1 = p["q"]
    k0, k1 = p["kv"]
    if family in ("w_qkv", "b_qkv"):
        idx = list(range(q0 * D, q1 * D)) + list(range((nq + k0) * D, (nq + k1) * D)) + \
            list(range((nq + nkv + k0) * D, (nq + nkv + k1) * D))
        return t[torch.tensor(idx)]
    if family == "w_o":
        return t[:, q0 * D:q1 * D]
    if family == "w_gu":
        # storage order of the engine: 64-row blocks [gate c | up c] (fused SwiGLU epilogue)
        f0, f1 = p["ffn"]
        blocks = []
        for a in range(f0, f1, 64):
            b = min(a + 64, f1)
            blocks += [t[a:b], t[F + a:F + b]]
        return torch.cat(blocks, dim=0)
    if family == "w_d":
        f0, f1 = p["ffn"]
        return t[:, f0:f1]
    if family == "lm_head":
        v0, v1 = p["vocab"]
        return t[v0:v1]
    return t  # replicated: norms, embedding


class ByteMemory:
    """Sparse byte-addressed memory: named buffers at fake base addresses."""

    def __init__(self):
        self.bufs: list[tuple[int, np.ndarray]] = []
        self._next = 1 << 40

    def alloc(self, nbytes: int) -> int:
        base = self._next
        self.bufs.append((base, np.zeros(nbytes, dtype=np.uint8)))
        self._next += ((nbytes + (1 << 20)) >> 20 << 20) + (1 << 30)
        return base

    def view(self, ptr: int, nbytes: int) -> np.ndarray:
        for base, arr in self.bufs:
            if base <= ptr and ptr + nbytes <= base + arr.size:
                return arr[ptr - base: ptr - base + nbytes]
        raise IndexError(f"address {ptr:#x}+{nbytes} is outside every buffer")

    def execute(self, items: np.ndarray) -> None:
        """Apply copy items (read everything first: items of one launch never alias)."""
        data = [self.view(int(s), int(n)).copy() for s, _, n, _ in items]
        for (s, d, n, _), blob in zip(items, data):
            self.view(int(d), int(n))[:] = blob


def expand_kv_moves(mem: "ByteMemory", moves: np.ndarray, dst_kv: int, dst_num_pages: int, dst_nkv: int,
                    layers: int, chunk: int) -> np.ndarray:
    """CPU restatement of tps_kv_move_items (csrc/copy.cu kv_move_items_kernel): every move
    (KV_MOVE_DTYPE record) becomes one copy item per (layer, k|v, valid page), page indices read
    from the page-table rows the move points at (here: in `mem`). Item order: move-major, then
    (layer * 2 + k|v), then page -- i.e. item index = first_item + lkv * n_pages + page."""
    out = []
    for m in moves:
        n_pages = int(m["n_pages"])
        sp = mem.view(int(m["src_pages"]), 4 * n_pages).view(np.int32)
        dp = mem.view(int(m["dst_pages"]), 4 * n_pages).view(np.int32)
        nh, snp, snkv = int(m["n_heads"]), int(m["src_num_pages"]), int(m["src_nkv"])
        for lkv in range(2 * layers):
            for p in range(n_pages):
                s = int(m["src_kv"]) + ((lkv * snp + int(sp[p])) * snkv + int(m["src_head"])) * chunk
                d = dst_kv + ((lkv * dst_num_pages + int(dp[p])) * dst_nkv + int(m["dst_head"])) * chunk
                out.append((s, d, nh * chunk, 0))
    return np.asarray(out, dtype=np.int64).reshape(-1, 4)
