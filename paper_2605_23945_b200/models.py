"""Executable decoder geometries and their canonical tensor-parallel partition.

The reference reduces a model to (layers, hidden, bytes/elem, bytes/layer)
(tpshift/cluster.py:19-49) and shards everything as contiguous hidden-dim
slices, rank r owning [r*D/tp, (r+1)*D/tp) (tpshift/reshard.py:25-43). Real
GQA decoders need a head-aware version of that rule; this module defines it,
and the weight reshard, the KV migration and the CPU oracle all follow it:

* KV heads are split contiguously when tp divides n_kv; otherwise (tp > n_kv,
  e.g. Qwen2.5-7B at TP8 with 4 KV heads) each KV head is replicated on
  m = tp / n_kv consecutive ranks and its G query heads are split into m
  contiguous parts, the first parts taking the remainder (7 -> 4 + 3).
* FFN columns and vocabulary rows are split contiguously (ShardLayout rule).
* Norm weights and the embedding table are replicated.
"""

from __future__ import annotations

from dataclasses import dataclass

from .cluster import ModelSpec
from .errors import ConfigError


@dataclass(frozen=True)
class DecoderGeometry:
    """A Llama / Qwen2-style decoder: RMSNorm, RoPE, GQA, SwiGLU."""

    name: str
    num_layers: int
    hidden: int
    n_q: int
    n_kv: int
    head_dim: int
    ffn: int
    vocab: int
    qkv_bias: bool
    rope_theta: float
    rms_eps: float = 1e-6
    bytes_per_elem: int = 2

    def __post_init__(self):
        if self.n_q % self.n_kv:
            raise ConfigError("n_q must be a multiple of n_kv")
        if self.head_dim not in (64, 128):
            raise ConfigError("head_dim must be 64 or 128")

    @property
    def group(self) -> int:
        return self.n_q // self.n_kv

    @property
    def qkv_rows(self) -> int:
        return (self.n_q + 2 * self.n_kv) * self.head_dim

    def layer_tensor_bytes(self) -> dict[str, int]:
        e, H, F, D = self.bytes_per_elem, self.hidden, self.ffn, self.head_dim
        out = {
            "w_qkv": self.qkv_rows * H * e,
            "w_o": H * self.n_q * D * e,
            "w_gu": 2 * F * H * e,
            "w_d": H * F * e,
            "ln1": H * e,
            "ln2": H * e,
        }
        if self.qkv_bias:
            out["b_qkv"] = self.qkv_rows * e
        return out

    @property
    def layer_param_bytes(self) -> int:
        return sum(self.layer_tensor_bytes().values())

    @property
    def kv_bytes_per_token(self) -> int:
        """Real GQA K+V bytes per token over all layers (unsharded)."""
        return 2 * self.num_layers * self.n_kv * self.head_dim * self.bytes_per_elem

    def model_spec(self) -> ModelSpec:
        """The reference's reduced ModelSpec for this geometry (cost-model view)."""
        return ModelSpec(name=self.name, num_layers=self.num_layers, hidden_dim=self.hidden,
                         bytes_per_elem=self.bytes_per_elem,
                         layer_param_bytes=self.layer_param_bytes)

    def check_tp(self, tp: int) -> None:
        if self.n_kv % tp and tp % self.n_kv:
            raise ConfigError(f"{self.name}: tp={tp} neither divides nor is a multiple of n_kv={self.n_kv}")
        if tp > self.n_kv and self.group < tp // self.n_kv:
            raise ConfigError(f"{self.name}: too few query heads per KV head for tp={tp}")
        if self.ffn % tp or self.vocab % tp:
            raise ConfigError(f"{self.name}: ffn and vocab must be divisible by tp={tp}")
        if (self.ffn // tp) % 64:
            raise ConfigError(f"{self.name}: ffn/tp must be a multiple of 64 (gate/up blocks)")


PRESETS: dict[str, DecoderGeometry] = {
    # BASELINE config 1: tiny GPT-style decoder (2 layers, d=256), same block family
    "tiny": DecoderGeometry("tiny", num_layers=2, hidden=256, n_q=4, n_kv=2, head_dim=64,
                            ffn=1024, vocab=4096, qkv_bias=True, rope_theta=10000.0),
    # config 2
    "qwen2.5-7b": DecoderGeometry("qwen2.5-7b", num_layers=28, hidden=3584, n_q=28, n_kv=4,
                                  head_dim=128, ffn=18944, vocab=152064, qkv_bias=True,
                                  rope_theta=1000000.0, rms_eps=1e-6),
    # config 3
    "llama3-8b": DecoderGeometry("llama3-8b", num_layers=32, hidden=4096, n_q=32, n_kv=8,
                                 head_dim=128, ffn=14336, vocab=128256, qkv_bias=False,
                                 rope_theta=500000.0, rms_eps=1e-5),
    # config 4
    "qwen2.5-32b": DecoderGeometry("qwen2.5-32b", num_layers=64, hidden=5120, n_q=40, n_kv=8,
                                   head_dim=128, ffn=27648, vocab=152064, qkv_bias=True,
                                   rope_theta=1000000.0, rms_eps=1e-6),
    # small GQA geometry used by GPU parity tests (head_dim 128, G=7 like Qwen2.5-7B)
    "mini-qwen": DecoderGeometry("mini-qwen", num_layers=2, hidden=512, n_q=14, n_kv=2,
                                 head_dim=128, ffn=1024, vocab=8192, qkv_bias=True,
                                 rope_theta=1000000.0),
    # small geometries with config 3's and config 4's head structure: Llama-3 (G=4, 8 KV
    # heads, no QKV bias: TP up to 8 without KV replication) and Qwen2.5-32B (G=5, 8 KV heads)
    "mini-llama": DecoderGeometry("mini-llama", num_layers=2, hidden=1024, n_q=8 * 4, n_kv=8,
                                  head_dim=32 * 4, ffn=2048, vocab=8192, qkv_bias=False,
                                  rope_theta=500000.0, rms_eps=1e-5),
    "mini-qwen32": DecoderGeometry("mini-qwen32", num_layers=2, hidden=640, n_q=40, n_kv=8,
                                   head_dim=128, ffn=1536, vocab=8192, qkv_bias=True,
                                   rope_theta=1000000.0),
}


def geometry(name: str) -> DecoderGeometry:
    try:
        return PRESETS[name]
    except KeyError:
        raise ConfigError(f"unknown model {name!r}; known: {', '.join(PRESETS)}") from None


@dataclass(frozen=True)
class RankShard:
    """What TP rank ``rank`` of a ``tp``-way group owns (global index ranges)."""

    tp: int
    rank: int
    q_heads: tuple[int, int]
    kv_heads: tuple[int, int]
    ffn: tuple[int, int]
    vocab: tuple[int, int]

    @property
    def n_q(self) -> int:
        return self.q_heads[1] - self.q_heads[0]

    @property
    def n_kv(self) -> int:
        return self.kv_heads[1] - self.kv_heads[0]

    @property
    def ffn_width(self) -> int:
        return self.ffn[1] - self.ffn[0]

    @property
    def vocab_width(self) -> int:
        return self.vocab[1] - self.vocab[0]


def rank_shard(geom: DecoderGeometry, tp: int, rank: int) -> RankShard:
    geom.check_tp(tp)
    if not 0 <= rank < tp:
        raise ConfigError(f"rank {rank} out of range for tp={tp}")
    G = geom.group
    if geom.n_kv % tp == 0:
        per = geom.n_kv // tp
        kv = (rank * per, (rank + 1) * per)
        q = (kv[0] * G, kv[1] * G)
    else:
        m = tp // geom.n_kv
        h, sub = divmod(rank, m)
        base, extra = divmod(G, m)
        sizes = [base + (1 if i < extra else 0) for i in range(m)]
        start = h * G + sum(sizes[:sub])
        q = (start, start + sizes[sub])
        kv = (h, h + 1)
    fw, vw = geom.ffn // tp, geom.vocab // tp
    return RankShard(tp=tp, rank=rank, q_heads=q, kv_heads=kv,
                     ffn=(rank * fw, (rank + 1) * fw), vocab=(rank * vw, (rank + 1) * vw))


GU_BLOCK = 64  # gate/up interleave block (rows)


# Sharded tensor families: (axis, full-coordinate ranges in shard storage order).
# axis 0 = rows of a row-major [rows][cols] tensor, axis 1 = columns.
def shard_ranges(geom: DecoderGeometry, family: str, sh: RankShard) -> tuple[int, list[tuple[int, int]]]:
    D = geom.head_dim
    q0, q1 = sh.q_heads
    k0, k1 = sh.kv_heads
    if family in ("w_qkv", "b_qkv"):
        kb = geom.n_q * D
        vb = kb + geom.n_kv * D
        return 0, [(q0 * D, q1 * D), (kb + k0 * D, kb + k1 * D), (vb + k0 * D, vb + k1 * D)]
    if family == "w_o":
        return 1, [(q0 * D, q1 * D)]
    if family == "w_gu":
        # interleaved 64-row blocks [gate c | up c]: one 128-row GEMM tile holds the gate
        # and up rows of the same 64 features, so SiLU(gate)*up fuses into its epilogue
        f0, f1 = sh.ffn
        out = []
        for a in range(f0, f1, GU_BLOCK):
            b = min(a + GU_BLOCK, f1)
            out += [(a, b), (geom.ffn + a, geom.ffn + b)]
        return 0, out
    if family == "w_d":
        return 1, [sh.ffn]
    if family == "lm_head":
        return 0, [sh.vocab]
    if family in ("ln1", "ln2", "ln_f", "embed"):
        return 0, [(0, full_shape(geom, family)[0])]
    raise ConfigError(f"unknown tensor family {family!r}")


def full_shape(geom: DecoderGeometry, family: str) -> tuple[int, ...]:
    H = geom.hidden
    return {
        "w_qkv": (geom.qkv_rows, H),
        "b_qkv": (geom.qkv_rows,),
        "w_o": (H, geom.n_q * geom.head_dim),
        "w_gu": (2 * geom.ffn, H),
        "w_d": (H, geom.ffn),
        "ln1": (H,),
        "ln2": (H,),
        "ln_f": (H,),
        "embed": (geom.vocab, H),
        "lm_head": (geom.vocab, H),
    }[family]


def shard_shape(geom: DecoderGeometry, family: str, sh: RankShard) -> tuple[int, ...]:
    full = full_shape(geom, family)
    axis, ranges = shard_ranges(geom, family, sh)
    width = sum(b - a for a, b in ranges)
    shape = list(full)
    shape[axis] = width
    return tuple(shape)


LAYER_FAMILIES = ("w_qkv", "b_qkv", "w_o", "w_gu", "w_d", "ln1", "ln2")
GLOBAL_FAMILIES = ("embed", "ln_f", "lm_head")


def layer_families(geom: DecoderGeometry) -> tuple[str, ...]:
    return tuple(f for f in LAYER_FAMILIES if f != "b_qkv" or geom.qkv_bias)


def rope_tables(geom: DecoderGeometry, max_pos: int):
    """fp32 cos/sin tables [max_pos][D/2] for rotate-half RoPE (computed in fp64)."""
    import numpy as np

    D = geom.head_dim
    inv = 1.0 / (geom.rope_theta ** (np.arange(0, D, 2, dtype=np.float64) / D))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
