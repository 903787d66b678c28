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
import gc
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
    "overhead_bytes": split-K partial bytes beyond one output, "n": launches}} plus "total"
    over one decode step's projections. Algorithmic bytes (SURVEY 8(d) units) = weight shard +
    activations read + one fp32 output row per batch row; the extra fp32 partials of a
    split-K launch (written, then read back by the consumer) are overhead, not algorithmic.
    """
    g = ex.geom
    lib = nat.lib()
    st = torch.cuda.current_stream()
    out = {}
    xs = {"w_qkv": ex.xn, "w_o": ex.attn, "w_gu": ex.xn, "w_d": ex.act}
    fams = [(f, [(l, f) for l in range(g.num_layers)]) for f in ("w_qkv", "w_o", "w_gu", "w_d")]
    fams.append(("lm_head", [(-1, "lm_head")] * max(1, g.num_layers // 4)))
    tot_ms = tot_b = tot_o = 0.0
    launches = 0
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
        byt = n * k * 2 + B * k * 2 + B * n * 4  # weights + activations + one fp32 output
        ovh = (s - 1) * B * n * 4  # the other split partials (written + read back: x2 on HBM)
        out[fam] = {"ms": ms, "bytes": byt, "overhead_bytes": ovh, "n": len(keys) if fam != "lm_head" else 1,
                    "splits": s}
        per_step = g.num_layers if fam != "lm_head" else 1
        tot_ms += ms * per_step
        tot_b += byt * per_step
        tot_o += ovh * per_step
        launches += per_step
    out["total"] = {"ms": tot_ms, "bytes": tot_b, "overhead_bytes": tot_o, "launches": launches,
                    "gbps": tot_b / tot_ms / 1e6}
    return out


def tail_probe(geom, tp: int, batches, ctx: int, peak_gbps: float, n: int = 30, gemv: bool = True) -> dict:
    """Post-switch tail steps (SURVEY 8(d) "tail = post-switch B <= 32"): one TP-`tp` rank alone on
    the device (loopback peer table, `loopback_rank`), graph-replayed steps at context `ctx` per
    batch, vs the rank's HBM floor = weight shards (linears + LM-head shard) + live K/V + new K/V
    at the measured copy peak. Returns {B: {"ms", "floor_ms", "frac", "kernels"}}; with `gemv`,
    buckets the warp-shuffle GEMV takes (<= tps_gemv_max_rows()) are also timed with every
    projection on it ("gemv_ms", "gemv_frac") -- the A/B behind executor.GEMV_ROWS."""
    from .kvcache import pages_for
    from .models import rank_shard
    from .shards import arena_layout
    maxb = max(batches)
    r, runner = loopback_rank(geom, tp, maxb, maxb, ctx + 256, maxb * pages_for(ctx + 256))
    slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(maxb)]
    sh = rank_shard(geom, tp, 0)
    lay = arena_layout(geom, sh)
    emb = geom.vocab * geom.hidden * 2
    w = lay.total_bytes - emb  # embedding rows are gathered, not streamed
    kv_tok = geom.num_layers * 2 * sh.n_kv * geom.head_dim * 2
    out = {}
    for B in batches:
        bk = r.executor.bucket(B)
        runner.set_rows(bk, slots[:B])
        r.slots.pos[:] = ctx
        ms = step_probe(runner, bk, n)
        byt = w + B * (ctx + 1) * kv_tok
        floor = byt / (peak_gbps * 1e9) * 1e3
        out[B] = {"ms": ms, "floor_ms": floor, "frac": floor / ms, "bytes": byt,
                  "gbps": byt / ms / 1e6, "frac_nominal_8tbps": byt / ms / 1e6 / 8000.0,
                  "kernels": runner.kernels_per_step(bk)}
        if gemv and bk <= nat.lib().tps_gemv_max_rows():
            default = r.executor.gemv_rows
            r.executor.gemv_rows = bk
            runner.graphs.pop(bk, None)  # recapture the bucket with the GEMV projections
            r.slots.pos[:] = ctx
            gms = step_probe(runner, bk, n)
            out[B].update({"gemv_ms": gms, "gemv_frac": floor / gms})
            r.executor.gemv_rows = default
            runner.graphs.pop(bk, None)
    del r, runner
    gc.collect()
    torch.cuda.empty_cache()
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


def _pav(y: np.ndarray, w: np.ndarray | None = None) -> np.ndarray:
    """Pool-adjacent-violators: the least-squares non-decreasing fit of y."""
    w = np.ones_like(y) if w is None else w
    vals, wts, cnt = [], [], []
    for yi, wi in zip(y, w):
        vals.append(float(yi))
        wts.append(float(wi))
        cnt.append(1)
        while len(vals) > 1 and vals[-2] > vals[-1]:
            v = (vals[-2] * wts[-2] + vals[-1] * wts[-1]) / (wts[-2] + wts[-1])
            wt, c = wts[-2] + wts[-1], cnt[-2] + cnt[-1]
            vals[-2:], wts[-2:], cnt[-2:] = [v], [wt], [c]
    return np.repeat(np.asarray(vals), cnt)


def monotone_table(table, passes: int = 4):
    """The Offline Profiler's measured table made physically monotone: a decode step cannot get
    faster with more context (same tp, batch) nor with more rows (same tp, context). Each
    measured point is a 60-step mean with ~1-3 % run-to-run noise (152 of 660 adjacent context
    pairs of the Qwen2.5-7B table decrease); least-squares isotonic fits along the context axis
    and then the batch axis, alternated, remove those inversions -- which otherwise surface as
    near-ties between neighbouring TP degrees that Algorithm 1 flips between. Prefill latencies
    (measured chunked-prefill steps) are kept. Grid, coverage and token cap are unchanged; the
    raw table stays the CSV of record."""
    from .latency import ProfilePoint, table_from_points
    pts = {(p.tp, p.batch, p.ctx_len): p.decode_latency for p in table.points}
    for _ in range(passes):
        for axis in (2, 1):
            groups = {}
            for k in pts:
                key = (k[0], k[1]) if axis == 2 else (k[0], k[2])
                groups.setdefault(key, []).append(k)
            for keys in groups.values():
                keys.sort(key=lambda k: k[axis])
                fit = _pav(np.array([pts[k] for k in keys]))
                for k, v in zip(keys, fit):
                    pts[k] = float(v)
    out = [ProfilePoint(p.tp, p.batch, p.ctx_len, pts[(p.tp, p.batch, p.ctx_len)], p.prefill_latency)
           for p in table.points]
    return table_from_points(out, table.token_cap)


def c_float(x: float):
    return ctypes.c_float(x)


def switch_probe(spec, geom, world, tp_to: int, n_samples: int, ctx: int, copy_mode: int = 0,
                 reps: int = 1, alias_replicas: bool = False, use_graphs: bool = True) -> dict:
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
        be = B200Backend(spec, geom, world, seed=0, alias_replicas=alias_replicas, use_graphs=use_graphs)
        be.capture_all(every_layout=True)   # what GlobalCoordinator does before a stage
        be.prepare_switch_items()
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
        marks = t.marks  # per rank: arrive, released, weights done, KV done, resumed
        t0 = min(be.start[r].elapsed_time(m[0]) for r, m in marks.items())
        t_rel = min(be.start[r].elapsed_time(m[1]) for r, m in marks.items())
        t_end = max(be.start[r].elapsed_time(m[4]) for r, m in marks.items())
        peer = max((v["nvlink"] for v in t.per_rank.values()), default=0)
        local = max((v["local"] for v in t.per_rank.values()), default=0)
        out.append({"weights_bytes": t.weight_bytes, "kv_bytes": t.kv_bytes, "nvlink_bytes": t.nvlink_bytes,
                    "local_bytes": t.local_bytes, "max_gpu_peer_bytes": peer, "max_gpu_local_bytes": local,
                    "copy_bytes": kbytes, "copy_kernel_ms": kms,
                    "copy_gbps": kbytes / (kms / 1e3) / 1e9, "switch_device_ms": t_end - t0,
                    "release_to_resume_ms": t_end - t_rel, "host_switch_s": t.host_s,
                    "host_plan_s": t.host_plan_s, "host_capture_s": t.host_capture_s,
                    "host_build_s": t.host_build_s, "copy_launches": len(be.copy_events)})
        del be
        gc.collect()  # backends hold reference cycles (runners <-> executors)
        torch.cuda.empty_cache()
    best = min(out, key=lambda d: d["copy_kernel_ms"])
    return best


def _start_event(be, r):
    e = torch.cuda.Event(enable_timing=True)
    e.record(be.stream(r))
    return e


# ------------------------------------------------------------------------------------------
# Offline Profiler on one B200 for every TP degree (tpshift/latency.py:229-250)
# ------------------------------------------------------------------------------------------

NVLINK_GBPS = 770.0       # measured peer-copy bandwidth per direction (B200_PROFILING.md)
NVLINK_HOP_S = 1.5e-6     # remote-store + release/acquire flag latency of one allreduce hop


def loopback_rank(geom, tp: int, max_batch: int, num_slots: int, max_len: int, kv_pages: int,
                  prefill_rows: int = 0, device="cuda:0", seed: int = 0):
    """One rank of a TP-`tp` group alone on the device: its peer table points at itself,
    so every allreduce push lands in its own receive area and every signal list holds its
    own counter tp times. The rank runs exactly the kernels, shapes and counter protocol
    of a real TP-`tp` rank; only the NVLink hop is missing (added back by the model in
    `nvlink_adjust`). Numerics are not meaningful -- this is a timing harness."""
    from .executor import GroupRunner
    from .group import build_rank
    r = build_rank(geom, tp, 0, max_batch, num_slots, max_len, device, seed=seed, kv_pages=kv_pages,
                   prefill_rows=prefill_rows)
    if r.comm is not None:
        r.comm.connect([r.comm.export()] * tp)
        r.comm.loopback = True
    return r, GroupRunner([r.executor])


def nvlink_adjust(geom, tp: int, batch: int) -> float:
    """Seconds per decode step that a real TP group adds over the loopback rank: for each
    of the 2L allreduces one NVLink hop plus the bytes this rank pushes to its tp-1 peers."""
    if tp == 1:
        return 0.0
    from .executor import FUSE_ROWS, FUSE_SOURCES, LL_CLUSTER_MIN_TP, LL_CLUSTER_ROWS, LL_EPILOGUE_ROWS
    # B <= 64: LL pairs (8 B per element) of the summed row (cluster-reduced epilogue or
    # reduce-push); else B <= 16: of every split partial (<= FUSE_SOURCES slots per group);
    # larger: the summed fp32 row (reduce-push)
    if batch <= min(LL_CLUSTER_ROWS, FUSE_ROWS) and tp >= LL_CLUSTER_MIN_TP:
        per_row = geom.hidden * 8 * (tp - 1)
    elif batch <= LL_EPILOGUE_ROWS:
        per_row = geom.hidden * 8 * (tp - 1) * max(1, FUSE_SOURCES // tp)
    elif batch <= FUSE_ROWS:
        per_row = geom.hidden * 8 * (tp - 1)
    else:
        per_row = geom.hidden * 4 * (tp - 1)
    return 2 * geom.num_layers * (NVLINK_HOP_S + batch * per_row / (NVLINK_GBPS * 1e9))


def profile_rank(geom, tp: int, token_cap: int, max_ctx: int, batches=None, lengths=None,
                 prefill_rows: int = 512, time_budget_s: float = 900.0, log=None):
    """Measured ProfilePoints of one TP degree on this device.

    decode: the reference's protocol (tpshift/latency.py:229-250) on the real engine --
    `batch` sequences at context L, 60 graph-replayed steps (contexts grow by one per
    step), mean step time, plus `nvlink_adjust` for tp > 1.
    prefill: the chunked prefill this engine runs (prompt positions through the decode
    kernels, `prefill_rows` rows per step): ceil(batch * (L - 1) / rows) steps, each
    timed at the mean context L / 2 (interpolated over a few measured contexts)."""
    from .latency import ProfilePoint
    batches = batches or [b for b in profile_batches()]
    lengths = lengths or [l for l in profile_lengths() if l + PROFILE_DECODE_STEPS + 2 <= max_ctx]
    grid = [(b, l) for b in batches for l in lengths if b * l <= token_cap]
    max_b = max(b for b, _ in grid)
    need = max(b * pages_for_tokens(l + PROFILE_DECODE_STEPS + 2) for b, l in grid)
    r, runner = loopback_rank(geom, tp, max_b, max_b, max_ctx, need, prefill_rows=prefill_rows)
    ex = r.executor
    st = r.slots
    t0 = time.perf_counter()
    dec = {}
    for b, l in grid:
        if time.perf_counter() - t0 > time_budget_s:
            break
        ppl = pages_for_tokens(l + PROFILE_DECODE_STEPS + 2)
        pt = torch.arange(b * ppl, dtype=torch.int32).view(b, ppl)
        st.page_table[:b, :ppl].copy_(pt)
        st.pos[:b] = l - 1
        bk = ex.bucket(b)
        runner.set_rows(bk, list(range(b)))
        ms = step_probe(runner, bk, PROFILE_DECODE_STEPS)
        dec[(b, l)] = ms / 1e3 + nvlink_adjust(geom, tp, b)
        if log:
            log(f"tp={tp} B={b} L={l}: {ms:.3f} ms")
    # prefill step time at `prefill_rows` rows vs context (rows spread over samples)
    pf = {}
    R = prefill_rows
    for ctx in [c for c in (64, 512, 2048, 8192) if c + 2 <= max_ctx]:
        nb = max(1, min(max_b, R))
        ppl = pages_for_tokens(ctx + 2)
        if nb * ppl > need:
            nb = max(1, need // ppl)
        pt = torch.arange(nb * ppl, dtype=torch.int32).view(nb, ppl)
        st.page_table[:nb, :ppl].copy_(pt)
        rs = torch.tensor([i % nb for i in range(R)], dtype=torch.int32)
        rp = torch.tensor([min(ctx, (i // nb) + ctx - (R // nb)) for i in range(R)], dtype=torch.int32)
        ex.set_prefill_rows(rs, rp)
        key = ("prefill", R)
        if key not in runner.graphs:
            runner._capture_key(key, lambda s_, rr=runner: rr._issue_prefill(R, s_))
        g = runner.graphs[key]
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = _events()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        pf[ctx] = e0.elapsed_time(e1) / 5 / 1e3 + nvlink_adjust(geom, tp, min(R, 64))
        if log:
            log(f"tp={tp} prefill step R={R} ctx={ctx}: {pf[ctx] * 1e3:.3f} ms")
    cs = np.array(sorted(pf), dtype=float)
    ts = np.array([pf[c] for c in sorted(pf)], dtype=float)
    pts = []
    for (b, l), d in dec.items():
        steps = -(-b * max(1, l - 1) // R)
        pts.append(ProfilePoint(tp, b, l, d, float(steps * np.interp(l / 2, cs, ts))))
    del runner, r
    gc.collect()
    torch.cuda.empty_cache()
    return pts


def pages_for_tokens(n: int) -> int:
    from .kvcache import PAGE
    return -(-n // PAGE)


def profile_b200(geom, tps=(1, 2, 4, 8), token_cap: int = 1 << 20, max_ctx: int = 16384 + 128,
                 time_budget_s: float = 900.0, log=None):
    """ProfileTable (the reference's CSV schema) measured on this B200 for every TP degree."""
    pts = []
    for tp in tps:
        geom.check_tp(tp)
        pts += profile_rank(geom, tp, token_cap, max_ctx, time_budget_s=time_budget_s / len(tps), log=log)
    keep = {}
    for p in pts:
        keep.setdefault((p.tp, p.batch), []).append(p)
    pts = [p for v in keep.values() if len(v) >= 2 for p in v]
    return table_from_points(pts, token_cap)
