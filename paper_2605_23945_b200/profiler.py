"""Offline Profiler on B200 (tpshift/latency.py:189-250) and kernel probes.

OfflineProfiler measures real decode-step latencies of the Infer Executor on
the reference's (tp, batch, ctx_len) grid (batch * ctx <= T_cap): for each
point, `batch` dummy sequences are placed at context ctx_len and the mean of
a 60-step graph-replayed window is recorded, exactly the reference's
protocol (decode window of PROFILE_DECODE_STEPS rounds whose aggregate tokens
grow by `batch` per step). Prefill on this engine runs through the decode
path, so its latency at (B, L) is the integral of the measured decode curve
over contexts 1..L-1. The result is a ProfileTable in the reference's CSV
schema that `fit_predictor` turns into the Latency Predictor.

`gemm_probe` / `step_probe` are the live roofline measurements bench.py reports.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _native as nat
from .executor import GroupRunner, InferExecutor
from .group import admit
from .latency import PROFILE_DECODE_STEPS, ProfilePoint, profile_batches, profile_lengths, table_from_points


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def gemm_probe(ex: InferExecutor, B: int, reps: int = 2) -> dict:
    """Time every projection family at batch B over all layers (working set >> L2).

    Returns {family: {"ms": avg launch ms, "bytes": algorithmic bytes per launch,
    "n": launches}} plus "total" over one decode step's projections. Algorithmic
    bytes = weight shard + activations read + fp32 partials written.
    """
    g = ex.geom
    lib = nat.lib()
    st = torch.cuda.current_stream()
    out = {}
    xs = {"w_qkv": ex.xn, "w_o": ex.attn, "w_gu": ex.xn, "w_d": ex.act}
    fams = [(f, [(l, f) for l in range(g.num_layers)]) for f in ("w_qkv", "w_o", "w_gu", "w_d")]
    fams.append(("lm_head", [(-1, "lm_head")] * max(1, g.num_layers // 4)))
    tot_ms = tot_b = 0.0
    for fam, keys in fams:
        x = xs.get(fam, ex.xn)
        w0 = ex.w[keys[0]]
        n, k = w0.shape
        s = lib.tps_linear_splits(n, k, B)
        for _ in range(2):  # warm
            nat.check(lib.tps_linear(w0.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                     ex.ws.data_ptr(), s, st.cuda_stream))
        e0, e1 = _events()
        e0.record(st)
        for _ in range(reps):
            for key in keys:
                w = ex.w[key]
                nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                         ex.ws.data_ptr(), s, st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        nl = reps * len(keys)
        ms = e0.elapsed_time(e1) / nl
        byt = n * k * 2 + B * k * 2 + s * B * n * 4  # weights + activations + fp32 split partials
        out[fam] = {"ms": ms, "bytes": byt, "n": len(keys) if fam != "lm_head" else 1, "splits": s}
        per_step = g.num_layers if fam != "lm_head" else 1
        tot_ms += ms * per_step
        tot_b += byt * per_step
    out["total"] = {"ms": tot_ms, "bytes": tot_b, "gbps": tot_b / tot_ms / 1e6}
    return out


def step_probe(runner: GroupRunner, B: int, n: int = 20) -> float:
    """Mean graph-replayed decode-step time (ms) for bucket B with current row binding."""
    if B not in runner.graphs:
        runner.capture(B)
    runner.step(B, 2)
    e0, e1 = _events()
    st = torch.cuda.current_stream()
    e0.record(st)
    runner.step(B, n)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


class OfflineProfiler:
    """Measure the (tp, batch, ctx) decode-latency grid of a rank group on this device."""

    def __init__(self, runner: GroupRunner, ranks, token_cap: int):
        self.runner = runner
        self.ranks = ranks
        self.token_cap = token_cap

    def grid(self, tp: int, max_batch: int, max_ctx: int) -> list[tuple[int, int, int]]:
        return [(tp, b, l) for b in profile_batches() for l in profile_lengths()
                if b * l <= self.token_cap and b <= max_batch and l + PROFILE_DECODE_STEPS <= max_ctx]

    def measure_point(self, B: int, L: int) -> float:
        """Mean step latency (s) over the reference's 60-step window starting at context L."""
        ex = self.ranks[0].executor
        slots = list(range(B))
        bk = ex.bucket(B)
        for r in self.ranks:
            r.slots.pos[:B] = L - 1  # contexts of length L (KV contents do not affect timing)
        self.runner.set_rows(bk, slots)
        return step_probe(self.runner, bk, PROFILE_DECODE_STEPS) / 1e3

    def run(self, tp: int, max_batch: int, max_ctx: int, time_budget_s: float = 600.0):
        t0 = time.perf_counter()
        pts = []
        by_b: dict[int, list[tuple[int, float]]] = {}
        for _, b, l in self.grid(tp, max_batch, max_ctx):
            if time.perf_counter() - t0 > time_budget_s:
                break
            by_b.setdefault(b, []).append((l, self.measure_point(b, l)))
        for b, curve in by_b.items():
            ls = np.array([c[0] for c in curve], dtype=float)
            ys = np.array([c[1] for c in curve], dtype=float)
            for l, y in curve:
                # prefill through the decode path: sum of step times over contexts 1..l-1
                xs = np.arange(1, l, dtype=float)
                pre = float(np.interp(xs, ls, ys).sum()) if l > 1 else y
                pts.append(ProfilePoint(tp, b, l, y, pre))
        keep = {}
        for p in pts:
            keep.setdefault((p.tp, p.batch), []).append(p)
        pts = [p for v in keep.values() if len(v) >= 2 for p in v]
        return table_from_points(pts, self.token_cap)


def c_float(x: float):
    return ctypes.c_float(x)


def switch_probe(spec, geom, world, tp_to: int, n_samples: int, ctx: int, copy_mode: int = 0,
                 reps: int = 1) -> dict:
    """Switch Executor microbench (BASELINE config 5): one real switch of a running decode.

    Builds the layout (spec.initial_tp, world), places `n_samples` live samples at
    context `ctx` (prompt = spec.prompt_len, the rest generated; KV contents are
    whatever the pages hold -- the copy is byte-exact regardless), places them
    with assign_merged_groups exactly as a committed switch does and executes the
    weight reshard + KV-page + history pulls to TP=tp_to. Returns bytes moved and
    the device time between the first and last copy event of the switch (the two
    device barriers excluded), per stream-ordered phase.
    """
    from .controller import assign_merged_groups
    from .coordinator import B200Backend
    from .workload import BatchStatus, Sample

    out = []
    for _ in range(reps):
        be = B200Backend(spec, geom, world, seed=0)
        lay = be.layout
        samples = {g: [] for g in range(lay.dp)}
        prompt = torch.zeros(spec.prompt_len, dtype=torch.int32)
        for i in range(n_samples):
            g = i % lay.dp
            grp = be.group_ranks(g)
            if not grp:
                continue
            slot = admit(grp, i, prompt, max_ctx=be.max_len)
            be.slot_of[i] = slot
            for r in grp:
                r.slots.pos[slot] = ctx - 1
            samples[g].append(Sample(id=i, prompt_len=spec.prompt_len, target_response_len=spec.l_max,
                                     generated_len=ctx - spec.prompt_len, intra_dp_group=g))
        statuses = [BatchStatus(0, g, tuple(v)) for g, v in samples.items()]
        merged = assign_merged_groups(statuses, tp_to, spec.cluster)
        for r in world.local_ranks:
            torch.cuda.synchronize(world.devices[r])
        be.copy_mode = copy_mode
        be.copy_events = []
        be.start = {r: _start_event(be, r) for r in world.local_ranks}
        be._execute_switch(tp_to, merged)
        t = be.switches[-1]
        for r in world.local_ranks:
            torch.cuda.synchronize(world.devices[r])
        # copy-kernel device time (launches of one stream are serial; a virtual world
        # runs every rank's pulls on the one device)
        kms = sum(e0.elapsed_time(e1) for e0, _, e1 in be.copy_events)
        kbytes = sum(nb for _, nb, _ in be.copy_events)
        marks = t.marks
        t0 = min(be.start[r].elapsed_time(m[0]) for r, m in marks.items())
        t_end = max(be.start[r].elapsed_time(m[3]) for r, m in marks.items())
        out.append({"weights_bytes": t.weight_bytes, "kv_bytes": t.kv_bytes, "nvlink_bytes": t.nvlink_bytes,
                    "local_bytes": t.local_bytes, "copy_bytes": kbytes, "copy_kernel_ms": kms,
                    "copy_gbps": kbytes / (kms / 1e3) / 1e9, "switch_device_ms": t_end - t0,
                    "host_plan_s": t.host_plan_s, "host_capture_s": t.host_capture_s,
                    "host_build_s": t.host_build_s, "copy_launches": len(be.copy_events)})
        del be
        torch.cuda.empty_cache()
    best = min(out, key=lambda d: d["copy_kernel_ms"])
    return best


def _start_event(be, r):
    e = torch.cuda.Event(enable_timing=True)
    e.record(be.stream(r))
    return e
