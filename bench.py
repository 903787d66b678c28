"""Benchmark: rollout time to the last finished sample (BASELINE.json metric) on B200.

Workload (BASELINE config 2, weak-scaled): Qwen2.5-7B-shaped random-init bf16
decoder, 64 samples per GPU (512 at 8 GPUs), 512-token synthetic prompts,
response lengths from the reference's long-tail mixture rescaled to an 8K
cap (seed 4), start at TP1/DP=N, Algorithm 1 switching over the TP degrees
that divide N. One "step" = one whole generation stage (prefill through the
decode path + decode to the last sample), run by the Global Coordinator.

  value      device-clock rollout seconds (CUDA events; prompts resident in HBM;
             max over ranks = the node's last completion), mean over K stages
  e2e        the same stage through the public API with prompts copied from
             pinned host memory and every sample's tokens copied back, host
             wall clock (includes launch/host overheads)
  roofline   dominant kernel = the tcgen05 projection GEMM, bytes/launch over
             CUDA-event time, per batch bucket, weighted by the stage's rounds
  cpu_baseline  the CPU oracle (oracle/decoder_ref.py) on this host's cores at full
             depth: decode steps timed at B = 1, 8, 64 and composed over the stage's rounds
  tail       the post-switch TP8 tail (one loopback rank, B <= 32) vs its HBM floor, with
             the warp-shuffle GEMV form (csrc/gemv.cu) timed beside the default at B <= 4
  gemv_stage the same stage with buckets of <= 4 rows on that GEMV (N=1, run last)

`--impl reference` times the reference-side CPU path (the oracle port) instead.
Run: python bench.py [--gpus N --steps K --warmup W]; N>1 under torchrun.
"""

from __future__ import annotations

import argparse
import dataclasses
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "rollout time to last sample (s) on 8xB200; switch reshard+KV-migrate GB/s"
UNIT = "s"
NOMINAL_HBM_GBPS = 8000.0  # B200 HBM3e nominal; SURVEY 8(d) asks for the fraction of both peaks


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--per-gpu-batch", type=int, default=64)
    ap.add_argument("--l-max", type=int, default=8192)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-switch", action="store_true")
    ap.add_argument("--static-tps", default="all",
                    help="N>1: also time the stage at these fixed TP degrees (default: every TP degree dividing N)")
    ap.add_argument("--no-tail", action="store_true")
    ap.add_argument("--no-gemv-ab", action="store_true",
                    help="N=1: skip the stage re-run with the tail buckets (<= 4 rows) on the warp-shuffle GEMV")
    ap.add_argument("--tp-list", default="", help="Algorithm 1 candidates (default: 1 and N, BASELINE config 2)")
    ap.add_argument("--initial-tp", type=int, default=1, help="starting TP degree (config 4 starts at TP2)")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--virtual", type=int, default=0,
                    help="run an N-rank virtual world on this one GPU (every rank shares the device: a "
                         "functional / memory run of a multi-GPU config, not a throughput number)")
    ap.add_argument("--alias-replicas", action="store_true",
                    help="with --virtual: DP replicas of a TP rank share one weight arena")
    return ap.parse_args()


def peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def build_spec(args, gpus):
    from paper_2605_23945_b200.config import build_scenario, load_config
    from paper_2605_23945_b200.controller import ControllerParams
    from paper_2605_23945_b200.models import geometry
    from paper_2605_23945_b200.workload import LengthDistribution
    import dataclasses
    cfg = load_config("b200")
    geom = geometry(args.model)
    cluster = dataclasses.replace(cfg.cluster, gpus_per_node=gpus)
    # BASELINE config 2 switches TP1/DP8 -> TP8/DP1: candidates {1, N}; --tp-list widens it
    # (config 3's multi-stage TP1 -> 2 -> 4 -> 8)
    want = [int(x) for x in getattr(args, "tp_list", "").split(",") if x] or \
        sorted({int(getattr(args, "initial_tp", 1) or 1), gpus})
    ctl = ControllerParams(tp_list=tuple(t for t in want if gpus % t == 0 and _tp_ok(geom, t)),
                           eval_interval=cfg.controller.eval_interval, chunk_steps=cfg.controller.chunk_steps)
    init_tp = int(getattr(args, "initial_tp", 1) or 1)
    if gpus % init_tp:
        init_tp = 1
    spec = build_scenario(cfg, prompt_len=args.prompt_len, global_batch=args.per_gpu_batch * gpus,
                          l_max=args.l_max, initial_tp=init_tp, seed=args.seed, controller=ctl)
    spec = dataclasses.replace(spec, model=geom.model_spec(), cluster=cluster,
                               distribution=LengthDistribution.default().scaled_to_cap(args.l_max))
    return spec, geom


def _tp_ok(geom, tp):
    try:
        geom.check_tp(tp)
        return True
    except Exception:
        return False


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        load = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


class CpuOracleSteps:
    """The CPU oracle (oracle/decoder_ref.py, vectorised over rows) at FULL depth: every layer,
    the real vocabulary, random bf16-valued weights (seeded torch CPU generator).
    `measure()` -> {"steps": {B: seconds of one decode step at context ctx}, "prefill64_s":
    seconds of a 64-token prefill chunk of one sample}.

    Timing only: every layer references one random layer's tensors (the same arithmetic and
    the same memory-to-core traffic per layer -- each layer's 1.9 GB of fp32 weights is far
    larger than the host caches -- in 1/L of the host memory and generation time), the LM head
    shares the embedding's tensor, and the rows of a step share one sample's cache."""

    def __init__(self, geom, threads: int, ctx: int = 2048, batches=(1, 8, 64)):
        from oracle.decoder_ref import OracleDecoder
        torch.set_num_threads(threads)
        t0 = time.perf_counter()
        g = torch.Generator().manual_seed(0)
        H, D, F, V = geom.hidden, geom.head_dim, geom.ffn, geom.vocab

        def rnd(*shape):
            return (torch.randn(*shape, generator=g) * 0.02).bfloat16().float()

        emb = rnd(V, H)
        W = {(-1, "embed"): emb, (-1, "ln_f"): torch.ones(H), (-1, "lm_head"): emb}
        one = {"w_qkv": rnd(geom.qkv_rows, H), "w_o": rnd(H, geom.n_q * D), "w_gu": rnd(2 * F, H),
               "w_d": rnd(H, F), "ln1": torch.ones(H), "ln2": torch.ones(H)}
        if geom.qkv_bias:
            one["b_qkv"] = rnd(geom.qkv_rows)
        for l in range(geom.num_layers):
            for k, v in one.items():
                W[(l, k)] = v
        geo = dict(num_layers=geom.num_layers, hidden=H, n_q=geom.n_q, n_kv=geom.n_kv, head_dim=D, ffn=F,
                   vocab=V, qkv_bias=geom.qkv_bias, rope_theta=geom.rope_theta, rms_eps=geom.rms_eps)
        self.orc = OracleDecoder(geo, W, tp=1, round_bf16=True, max_len=ctx + 8)
        self.orc.step([1], [ctx - 1], [0])  # allocates the shared cache
        self.ctx, self.batches = ctx, batches
        self.setup_s = time.perf_counter() - t0

    def measure(self) -> dict:
        t1 = time.perf_counter()
        self.orc.prefill(list(range(64)), sample=1, start=0)
        pre = time.perf_counter() - t1
        steps = {}
        for B in self.batches:
            t1 = time.perf_counter()
            self.orc.step([1] * B, [self.ctx - 1] * B, [0] * B)
            steps[B] = time.perf_counter() - t1
        return {"steps": steps, "prefill64_s": pre, "setup_s": self.setup_s, "ctx": self.ctx}


def cpu_decode_steps(geom, threads: int, ctx: int = 2048) -> dict:
    return CpuOracleSteps(geom, threads, ctx).measure()


def active_histogram(rep) -> dict[int, int]:
    """Rounds per active-sample count (whole node) from a SimReport's step blocks."""
    hist = {}
    for nr in rep.node_reports:
        for ev in nr["events"]:
            if ev["type"] == "step-block":
                lo, hi = (int(x) for x in ev["detail"].split("=")[1].split(".."))
                hist[ev["active"]] = hist.get(ev["active"], 0) + (hi - lo)
    return hist


def cpu_stage_estimate(spec, steps: dict, hist: dict[int, int]) -> float:
    """Stage seconds on the CPU oracle: every decode round at its active batch (measured
    full-depth step times, piecewise-linear in B between the measured batches, proportional to
    B beyond the largest) + the prompts' prefill at the measured 64-token chunk rate."""
    bs = sorted(steps["steps"])
    ys = [steps["steps"][b] for b in bs]

    def t(B):  # beyond the largest measured batch (N > 1 stages): proportional to the rows
        return float(np.interp(B, bs, ys)) if B <= bs[-1] else ys[-1] * B / bs[-1]
    dec = sum(n * t(B) for B, n in hist.items())
    pre = spec.global_batch * (spec.prompt_len / 64.0) * steps["prefill64_s"]
    return dec + pre


def cpu_switch_copy(geom, samples: int, ctx: int, threads: int, reps: int = 3, verify: bool = False) -> dict:
    """SURVEY 8(d) CPU baseline (ii) for the switch: BASELINE config 5's microbench switch
    (TP1/DP2 -> TP2/DP1, `samples` live samples at context `ctx`) as host copies with torch on
    this host's cores. Weights: the Switch Executor's own pull plan (`plan_weight_pulls`, the
    canonical slices of tpshift/reshard.py:25-43) executed piece by piece as byte-slice copies
    between host arenas (both old replicas hold identical bytes: one host arena stands for both).
    KV: every sample's pages gathered from its old group's pool and scattered into the new
    ranks' pools with the rank's KV heads ([2L][pages][n_kv][64][D] bf16, the engine's layout),
    one torch index copy per (sample, target rank). Returns bytes, seconds and GB/s of each
    part, median over `reps` passes (`verify`: also the host buffers, for the CPU test against
    the canonical shards of oracle/reshard_ref.py)."""
    from paper_2605_23945_b200.kvcache import PAGE, pages_for
    from paper_2605_23945_b200.models import rank_shard
    from paper_2605_23945_b200.shards import arena_layout
    from paper_2605_23945_b200.switch_executor import Layout, plan_weight_pulls
    torch.set_num_threads(threads)
    old, new = Layout(1, 2), Layout(2, 2)
    nsrc = arena_layout(geom, rank_shard(geom, 1, 0)).total_bytes
    src = torch.randint(0, 256, (nsrc,), dtype=torch.uint8, generator=torch.Generator().manual_seed(1)) \
        if verify else torch.ones(nsrc, dtype=torch.uint8)
    plans = [plan_weight_pulls(geom, old, new, r).arrays() for r in range(2)]
    dsts = [torch.zeros(arena_layout(geom, rank_shard(geom, 2, r)).total_bytes, dtype=torch.uint8)
            for r in range(2)]
    wbytes = int(sum(int(p[3].sum()) for p in plans))
    t_ws = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for (_, so, do, nb), dst in zip(plans, dsts):
            for a, b, n in zip(so.tolist(), do.tolist(), nb.tolist()):
                dst[b:b + n].copy_(src[a:a + n])
        t_ws.append(time.perf_counter() - t0)
    t_w = statistics.median(t_ws)
    L, nkv, D = geom.num_layers, geom.n_kv, geom.head_dim
    npg = pages_for(ctx)
    per_group = -(-samples // 2)
    g = torch.Generator().manual_seed(2)
    pools = [torch.randint(-2 ** 15, 2 ** 15, (L, 2, per_group * npg, nkv, PAGE, D), dtype=torch.int16, generator=g)
             for _ in range(2)]
    hk = [rank_shard(geom, 2, r).kv_heads for r in range(2)]
    new_pools = [torch.zeros((L, 2, samples * npg, b - a, PAGE, D), dtype=torch.int16) for a, b in hk]
    kbytes = samples * L * 2 * npg * nkv * PAGE * D * 2
    t_kvs = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for i in range(samples):
            old_g, j = i % 2, i // 2  # sample i ran in old DP group i % 2
            sp = torch.arange(j * npg, (j + 1) * npg)
            dp = torch.arange(i * npg, (i + 1) * npg)
            for r, (a, b) in enumerate(hk):
                new_pools[r][:, :, dp] = pools[old_g][:, :, sp, a:b]
        t_kvs.append(time.perf_counter() - t0)
    t_kv = statistics.median(t_kvs)
    out = {"weights_bytes": wbytes, "weights_s": t_w, "weights_gbps": wbytes / t_w / 1e9,
           "weight_pieces": int(sum(len(p[3]) for p in plans)), "kv_bytes": kbytes, "kv_s": t_kv,
           "kv_gbps": kbytes / t_kv / 1e9, "gbps": (wbytes + kbytes) / (t_w + t_kv) / 1e9, "cores": threads,
           "reps": reps}
    if verify:
        out["arenas"] = (src, dsts, plans, pools, new_pools, hk)
    return out


def cpu_switch_baseline(model: str, threads: int, layers: int = 4, samples: int = 16, ctx: int = 4096) -> dict:
    """cpu_switch_copy on a bounded sample of config 5's microbench switch: the first `layers`
    layers of the model (embedding, LM head and norms included); GB/s is per byte moved."""
    import dataclasses as dc
    from paper_2605_23945_b200.models import geometry
    geom = dc.replace(geometry(model), num_layers=layers)
    r = cpu_switch_copy(geom, samples, ctx, threads)
    r["sample"] = (f"c5 switch TP1/DP2 -> TP2/DP1 of {model} truncated to {layers} layers (+ embedding / LM head), "
                   f"{samples} samples at ctx {ctx}: the executor's weight pull plan as torch byte-slice copies "
                   f"and KV page gather/scatter per (sample, rank), {threads} threads")
    return r


REF_INSTALL = os.path.join(HERE, "baseline", "_ref")  # the unmodified reference (pip --target, __graft_entry__.build)


def reference_package():
    """The unmodified reference package `tpshift` from baseline/_ref (installed from
    /root/reference by __graft_entry__.build(); it travels to the GPU box), or None."""
    if not os.path.isdir(os.path.join(REF_INSTALL, "tpshift")):
        return None
    if REF_INSTALL not in sys.path:
        sys.path.insert(0, REF_INSTALL)
    import tpshift
    return tpshift


def to_reference(T, x):
    """This package's decision-layer value as the reference's type (interop.to_reference)."""
    from paper_2605_23945_b200.interop import to_reference as conv
    return conv(T, x)


def decision_layer_timing(args) -> dict:
    """The reference's own CPU path, single-threaded Python (SURVEY 8(d) CPU baseline (i)):
    Algorithm 1 `evaluate` at B=512 (BASELINE config 2 on 8 GPUs, TP1/DP8, mid-stage) and one
    whole simulated stage `run` -- the restated tpshift code, bit-exact with the reference."""
    from paper_2605_23945_b200.cluster import ParallelConfig
    from paper_2605_23945_b200.controller import evaluate
    from paper_2605_23945_b200.engine import build_hardware_model, planner_view, run as sim_run
    from paper_2605_23945_b200.switchcost import CommGroupPool
    from paper_2605_23945_b200.workload import BatchStatus, Sample, sample_response_lengths
    ns = argparse.Namespace(model=args.model, per_gpu_batch=64, l_max=args.l_max, prompt_len=args.prompt_len,
                            seed=args.seed, tp_list="1,2,4,8", initial_tp=1)
    spec, geom = build_spec(ns, 8)
    table = measured_table(args.model)
    pred, _ = planner_view(spec, build_hardware_model(spec), table)
    lens = sample_response_lengths(spec.distribution, spec.global_batch, spec.seed)
    l_gen = 1000
    groups = {g: [] for g in range(8)}
    for i, t in enumerate(lens):
        if min(t, spec.l_max) > l_gen:
            groups[i % 8].append(Sample(id=i, prompt_len=spec.prompt_len, target_response_len=int(t),
                                        generated_len=l_gen, intra_dp_group=i % 8))
    st = [BatchStatus(node_id=0, group_index=g, samples=tuple(v)) for g, v in groups.items()]
    pool = CommGroupPool.fresh(spec.switch.comm_init_cost, warm=((1, 8),))
    cur = ParallelConfig.for_cluster(spec.cluster, 1)
    live = sum(len(v) for v in groups.values())
    evaluate(spec.controller, pred, pool, spec.switch, st, cur, spec.l_max, l_gen, spec.model, spec.cluster)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        evaluate(spec.controller, pred, pool, spec.switch, st, cur, spec.l_max, l_gen, spec.model, spec.cluster)
    ev = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    rep = sim_run(spec, table)
    run_s = time.perf_counter() - t0
    out = {"evaluate_ms": ev * 1e3, "evaluate_live_samples": live, "run_stage_s": run_s,
           "run_stage": f"c2 on 8 GPUs: {spec.global_batch} samples, tp_list (1,2,4,8), "
                        f"{rep.eval_count} evaluations", "cores": 1,
           "impl": "restated (paper_2605_23945_b200 decision layer, bit-exact with tpshift)"}
    T = reference_package()
    if T is None:
        out["reference_impl"] = {"unavailable": "baseline/_ref has no tpshift install"}
        return out
    # the same two calls through the UNMODIFIED reference (tpshift from baseline/_ref), same inputs
    rspec, rtab = to_reference(T, spec), to_reference(T, table)
    rpred = T.fit_predictor(rtab)  # the reference's own predictor fit of the same measured table
    rargs = [to_reference(T, spec.controller), rpred] + [to_reference(T, a) for a in (pool, spec.switch, st, cur)]
    rmod, rcl = to_reference(T, spec.model), to_reference(T, spec.cluster)
    T.evaluate(*rargs, spec.l_max, l_gen, rmod, rcl)
    t0 = time.perf_counter()
    for _ in range(reps):
        T.evaluate(*rargs, spec.l_max, l_gen, rmod, rcl)
    rev = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    rrep = T.run(rspec, rtab)
    rrun = time.perf_counter() - t0
    dec, rdec = (evaluate(spec.controller, pred, pool, spec.switch, st, cur, spec.l_max, l_gen, spec.model,
                          spec.cluster), T.evaluate(*rargs, spec.l_max, l_gen, rmod, rcl))
    out["reference_impl"] = {"evaluate_ms": rev * 1e3, "run_stage_s": rrun, "cores": 1,
                             "report_identical": rrep.to_json() == rep.to_json(),
                             "decision_identical": (dec.action, repr(dec.t_cur), repr(dec.t_best)) ==
                                                   (rdec.action, repr(rdec.t_cur), repr(rdec.t_best)),
                             "source": "tpshift (unmodified reference) from baseline/_ref"}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import paper_2605_23945_b200 as pkg  # noqa: F401
    from paper_2605_23945_b200.cache_manager import World
    from paper_2605_23945_b200.coordinator import GlobalCoordinator
    from paper_2605_23945_b200.profiler import gemm_probe

    gpus = args.virtual or max(1, args.gpus)
    world = World.virtual(args.virtual) if args.virtual else (World.from_env() if gpus > 1 else World.virtual(1))
    rank = world.local_ranks[0]
    dev = world.devices[rank]
    spec, geom = build_spec(args, gpus)
    table = measured_table(args.model)
    t_setup = time.perf_counter()
    coord = GlobalCoordinator(spec, geom, world, seed=0, table=table,
                              **({"alias_replicas": True} if args.alias_replicas else {}))
    setup_s = time.perf_counter() - t_setup
    for _ in range(args.warmup):
        coord.run()
    times, walls, launches, reports = [], [], 0, []
    world.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index or 0) as clk:
        for _ in range(args.steps):
            rep, meas = coord.run()
            reports.append(rep)
            times.append(rep.generation_time)
            walls.append(coord.last_wall_s)
            launches += coord.backend.kernels_launched
    torch.cuda.synchronize(dev)
    world.barrier()
    value = float(np.mean(times))
    rep = reports[-1]
    e2e = None
    if not args.no_e2e:
        coord.backend.host_io = True
        erep, _ = coord.run()
        be = coord.backend
        e2e = {"value": coord.last_wall_s, "unit": UNIT, "h2d_bytes_per_step": be.h2d_bytes,
               "d2h_bytes_per_step": be.d2h_bytes, "device_clock_s": erep.generation_time}
        coord.backend.host_io = False
    # ---- roofline of the dominant kernel (tcgen05 projection GEMM), weighted by the stage's rounds
    # at the initial layout (rounds after a switch run sharded GEMMs of another TP degree)
    coord.backend.reset(0)
    ex = coord.backend.ranks[rank].executor
    dp0 = gpus // spec.initial_tp
    hist, other_rounds = {}, 0
    for nr in rep.node_reports:
        for ev in nr["events"]:
            if ev["type"] == "step-block":
                lo, hi = (int(x) for x in ev["detail"].split("=")[1].split(".."))
                if ev["tp"] != spec.initial_tp:
                    other_rounds += hi - lo
                    continue
                bk = ex.bucket(min(ex.max_batch, -(-ev["active"] // dp0)))
                hist[bk] = hist.get(bk, 0) + (hi - lo)
    probes = {}
    for B in sorted(hist):
        probes[B] = gemm_probe(ex, B)["total"]
    w_rounds = sum(hist.values())
    g_ms = sum(probes[B]["ms"] * n for B, n in hist.items()) / w_rounds
    g_bytes = sum(probes[B]["bytes"] * n for B, n in hist.items()) / w_rounds
    g_ovh = sum(probes[B]["overhead_bytes"] * n for B, n in hist.items()) / w_rounds
    g_launch = probes[max(hist, key=hist.get)]["launches"]
    peak, peak_src = peaks()
    achieved = g_bytes / g_ms / 1e6
    switch = [s for nr in rep.node_reports for s in nr["switches"]]
    sw_gbps = [s.get("peer_gbps_per_gpu") for s in switch if s.get("peer_gbps_per_gpu")]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"c2-weak: {args.model}-shaped random-init, {args.per_gpu_batch} samples/GPU, "
                               f"prompt {args.prompt_len}, long-tail lengths capped at {args.l_max} (seed "
                               f"{args.seed}), start TP{spec.initial_tp}/DP{gpus // spec.initial_tp}, Algorithm 1 over tp_list "
                               f"{list(spec.controller.tp_list)}",
                   "model": args.model, "global_batch": spec.global_batch, "seq_len": args.prompt_len + args.l_max,
                   "parallelism": f"tp{spec.initial_tp}->adaptive,dp{gpus // spec.initial_tp}", "l2": "inputs > L2 (14.1 GB of weight shards streamed per step)",
                   "step": "one generation stage (prefill via decode path + decode to last sample)",
                   "predictor": "B200-measured profile table" if table is not None else "analytic b200.cfg"},
        "phases": stage_phases(rep, meas),
        "tokens_generated": rep.tokens_generated,
        "tokens_per_s": rep.tokens_generated / value,
        "switches": [{"from": s["from_tp"], "to": s["to_tp"], "round": s["round"],
                      "seconds": s["breakdown"]["total"], "release_to_resume_s": s.get("release_to_resume_s"),
                      "max_gpu_peer_bytes": s.get("max_gpu_peer_bytes"),
                      "max_gpu_local_bytes": s.get("max_gpu_local_bytes"),
                      "peer_gbps_per_gpu": s.get("peer_gbps_per_gpu"), "host_switch_s": s.get("host_switch_s"),
                      # the reference plan's volumes beside the executed bytes
                      "reference_plan_bytes_per_rank": {"weights": s.get("weight_plan_per_rank_bytes"),
                                                        "kv": (s.get("kv_plan") or {}).get("per_rank_bytes")}}
                     for s in switch],
        "switch_gbps": (sum(sw_gbps) / len(sw_gbps)) if sw_gbps else None,
        "switch_gbps_note": "max over GPUs of bytes pulled from peers / that GPU's barrier-release -> resume "
                            "window (SURVEY 8(d)); local copies reported separately",
        "wall_s_per_step": float(np.mean(walls)),
        "setup_s": setup_s,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "kernel": "gemm_swapab_kernel (tcgen05)",
                     "peak_source": peak_src, "nominal_peak": NOMINAL_HBM_GBPS,
                     "frac_nominal": achieved / NOMINAL_HBM_GBPS,
                     "algorithmic_bytes_per_launch": g_bytes / g_launch, "launches_per_step": g_launch,
                     "split_partial_overhead_bytes_per_step": g_ovh,
                     "bytes_note": "algorithmic = weight shard + activations + one fp32 output row per batch row "
                                   "(SURVEY 8(d)); the other split-K partials are overhead (written and read "
                                   "back once more), excluded from achieved",
                     "per_bucket": {str(B): {"gbps": probes[B]["gbps"], "rounds": hist[B]} for B in sorted(hist)},
                     "rounds_at_other_tp": other_rounds},
        "clocks": clk.summary(),
        "peak_hbm_gb": torch.cuda.max_memory_allocated(dev) / 2 ** 30,
    }
    if args.virtual:
        line["virtual_world"] = (f"{args.virtual} ranks on one GPU (functional / memory run: every rank's kernels "
                                 f"share the device, so times are not N-GPU times)")
    if e2e:
        line["e2e"] = e2e
    if table is not None:
        # the Offline Profiler's prediction of this same stage: the reference engine loop replayed
        # over the measured table (SURVEY §8(f)2 predictor-error target: <= 8 %)
        from paper_2605_23945_b200.engine import TableBackend, run as sim_run
        pred = sim_run(spec, table, TableBackend(spec, table)).generation_time
        line["predicted"] = {"value": pred, "unit": UNIT, "rel_error": (pred - value) / value,
                             "source": "reference engine loop over presets/b200_<model>_profile.csv"}
    if gpus == 1 and spec.initial_tp == 1 and not line["switches"]:
        line["stage_roofline"] = stage_roofline(spec, geom, line["phases"]["decode_s"], peak)
    tr = traffic_record()
    if tr:
        line["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
        line["roofline"]["traffic_note"] = tr["note"]
    if gpus > 1 and args.static_tps:
        # the north-star comparison: the same stage at a fixed TP (no switching), same engine
        line["fixed_tp"] = {}
        fixed = [t for t in (1, 2, 4, 8) if t <= gpus] if args.static_tps == "all" else \
            [int(x) for x in args.static_tps.split(",")]
        for tp in fixed:
            if gpus % tp or not _tp_ok(geom, tp):
                continue
            # discard the previous backend: peers' mappings of its buffers are closed on every rank
            # before any rank frees them (CUDA IPC), then the memory goes back to the device
            torch.cuda.synchronize(dev)
            world.barrier()
            world.close_peers()
            world.barrier()
            ex = coord = None
            gc.collect()  # executors / runners / comms form reference cycles
            torch.cuda.empty_cache()
            sspec = dataclasses.replace(spec, mode="static", initial_tp=tp)
            coord = GlobalCoordinator(sspec, geom, world, seed=0, table=table,
                                      **({"alias_replicas": True} if args.alias_replicas else {}))
            coord.run()
            srep, _ = coord.run()
            line["fixed_tp"][str(tp)] = srep.generation_time
        if line["fixed_tp"]:
            best = min(line["fixed_tp"], key=line["fixed_tp"].get)
            line["adaptive_vs_best_fixed"] = {"adaptive_s": value, "best_fixed_tp": int(best),
                                              "best_fixed_s": line["fixed_tp"][best],
                                              "speedup": line["fixed_tp"][best] / value}
        line["active_gpus"] = sorted(world.devices[r].index or 0 for r in world.local_ranks) \
            if not world.distributed else list(range(gpus))
    if rank == 0 and gpus == 1 and not args.no_switch:
        try:
            line["switch_microbench"] = switch_microbench(args, peak)
        except Exception as e:
            line["switch_microbench"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and gpus == 1 and not args.no_tail:
        # the post-switch tail (BASELINE config 2 ends at TP8): one TP8 rank alone on this GPU
        # (loopback peer table: same kernels and protocol, no NVLink hop), B <= 32
        from paper_2605_23945_b200.profiler import tail_probe
        try:
            tail = tail_probe(geom, 8, (1, 4, 16, 32), 4096, peak)
            line["tail"] = {"tp": 8, "ctx": 4096, "per_batch": {str(b): v for b, v in tail.items()},
                            "note": "TP8 rank with a looped-back peer table (no NVLink hop); floor = weight shard "
                                    "+ LM-head shard + live and new K/V at the measured copy peak; gemv_ms = the "
                                    "same step with every projection on the warp-shuffle GEMV (csrc/gemv.cu)"}
        except Exception as e:
            line["tail"] = {"error": f"{type(e).__name__}: {e}"}
    steps = None
    threads = args.cpu_threads or os.cpu_count()
    if rank == 0 and gpus == 1 and not args.no_cpu:
        try:
            steps = cpu_decode_steps(geom, threads, ctx=stage_mean_context(spec))
        except Exception as e:  # the bench line must still print
            steps = None
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"CPU oracle failed: {type(e).__name__}: {e}"}
    if rank == 0 and gpus == 1 and not args.no_cpu and steps is not None:
        est = cpu_stage_estimate(spec, steps, active_histogram(rep))
        depth = f"full depth ({geom.num_layers} layers"
        line["cpu_baseline"] = {
            "value": est, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"CPU oracle at {depth}, vocab {geom.vocab}, torch fp32 "
                       f"with bf16 rounding, {threads} threads): decode steps measured at B="
                       + ",".join(f"{b} ({t:.2f} s)" for b, t in steps["steps"].items())
                       + f" at ctx {steps['ctx']} (the stage's round-weighted mean context) and a 64-token "
                         f"prefill chunk ({steps['prefill64_s']:.2f} s); the stage = its "
                         f"{sum(active_histogram(rep).values())} rounds at their active batch "
                         f"(interpolated in B) + {spec.global_batch} prompts' prefill"),
            "measured_steps_s": {str(b): t for b, t in steps["steps"].items()}}
        try:
            line["cpu_baseline"]["decision_layer"] = decision_layer_timing(args)
        except Exception as e:
            line["cpu_baseline"]["decision_layer"] = {"error": f"{type(e).__name__}: {e}"}
        try:
            line["cpu_baseline"]["switch"] = cpu_switch_baseline(args.model, threads)
        except Exception as e:
            line["cpu_baseline"]["switch"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and gpus == 1 and not args.no_gemv_ab and not args.virtual:
        # last (it rebuilds the backend): the same stage with every bucket of <= 4 rows on the
        # warp-shuffle GEMV (csrc/gemv.cu) -- the stage-level A/B behind executor.GEMV_ROWS
        try:
            ex = be = None  # (drop this frame's handles on the first backend before rebuilding)
            line["gemv_stage"] = gemv_stage_ab(spec, geom, world, table, coord)
        except Exception as e:
            line["gemv_stage"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def gemv_stage_ab(spec, geom, world, table, coord) -> dict:
    from paper_2605_23945_b200 import executor as exmod
    from paper_2605_23945_b200.coordinator import GlobalCoordinator
    coord.backend = None
    del coord
    gc.collect()
    torch.cuda.empty_cache()
    old = exmod.GEMV_ROWS
    exmod.GEMV_ROWS = 4
    try:
        c2 = GlobalCoordinator(spec, geom, world, seed=0, table=table)
        c2.run()  # warm-up stage
        rep, _ = c2.run()
    finally:
        exmod.GEMV_ROWS = old
    return {"value": rep.generation_time, "unit": UNIT, "gemv_rows": 4,
            "note": "the same stage (one warm-up, one timed) with buckets of <= 4 rows on the warp-shuffle GEMV; "
                    "compare with `value`"}


def stage_mean_context(spec) -> int:
    """Round-weighted mean context of a stage's active samples (prompt + generated so far)."""
    from paper_2605_23945_b200.workload import sample_response_lengths
    lens = np.minimum(np.asarray(sample_response_lengths(spec.distribution, spec.global_batch, spec.seed)),
                      spec.l_max)
    r = np.arange(int(lens.max()))
    active = (lens[None, :] > r[:, None])
    ctx = (spec.prompt_len + r)[:, None] * active
    return int(round(float(ctx.sum() / max(1, active.sum())) / 64.0) * 64)


def stage_roofline(spec, geom, decode_s: float, peak_gbps: float) -> dict:
    """HBM floor of the stage's decode rounds on one GPU at TP1: every round streams all
    weight shards (linears + LM head) and every active sample's K/V (SURVEY §8(d) units)."""
    from paper_2605_23945_b200.workload import sample_response_lengths
    lens = np.asarray(sample_response_lengths(spec.distribution, spec.global_batch, spec.seed))
    lens = np.minimum(lens, spec.l_max)
    w = geom.num_layers * geom.layer_param_bytes + geom.vocab * geom.hidden * geom.bytes_per_elem
    kvpt = geom.kv_bytes_per_token
    rounds = int(lens.max())
    r = np.arange(rounds)
    active = (lens[None, :] > r[:, None]).sum(1)
    total = float(rounds * w + (kvpt * (spec.prompt_len + r) * active).sum())
    floor = total / (peak_gbps * 1e9)
    return {"decode_floor_s": floor, "decode_s": decode_s, "frac": floor / decode_s, "bytes": total,
            "rounds": rounds, "note": "weights + live K/V per round at the measured copy peak"}


def stage_phases(rep, meas) -> dict:
    """Where the (last timed) stage went: prefill, decode rounds, switches (device clock)."""
    pre = max((g["prefill"] or 0.0) for g in meas["groups"].values()) if meas["groups"] else 0.0
    sw = [s for nr in rep.node_reports for s in nr["switches"]]
    t_sw = sum(s["breakdown"]["total"] for s in sw)
    return {"prefill_s": pre, "switch_s": t_sw, "decode_s": rep.generation_time - pre - t_sw,
            "switches": len(sw)}


def measured_table(model: str):
    """The B200 Offline Profiler's table for this model (presets/b200_<model>_profile.csv,
    measured by tools/profile_b200.py): Algorithm 1's Latency Predictor is fitted to it.
    None (the analytic b200.cfg calibration) when the model has not been profiled. The measured
    points are made monotone in context and batch first (profiler.monotone_table)."""
    from paper_2605_23945_b200.latency import load_table
    from paper_2605_23945_b200.profiler import monotone_table
    path = os.path.join(HERE, "paper_2605_23945_b200", "presets", f"b200_{model}_profile.csv")
    return monotone_table(load_table(path)) if os.path.exists(path) else None


def traffic_record():
    """ncu DRAM traffic of the projection GEMM per launch (profiles/r2/ncu_traffic.json, from
    `ncu --set full` of one QKV / O / gate-up / down launch each at B=64, averaged like
    `achieved`); falls back to the round-1 single-launch record."""
    try:
        with open(os.path.join(HERE, "profiles", "r2", "ncu_traffic.json")) as fh:
            d = json.load(fh)["gemm_swapab_kernel"]
        return {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "note": d["note"]}
    except Exception:
        pass
    try:
        with open(os.path.join(HERE, "profiles", "r1", "ncu_traffic.json")) as fh:
            d = json.load(fh)["gemm_swapab_kernel"]
        return {"dram_bytes_per_launch": d["dram_bytes"],
                "note": f"ncu dram read+write of one launch ({d['launch']}) vs its {d['algorithmic_bytes']} "
                        f"algorithmic bytes; profiles/r1/ncu_traffic.json"}
    except Exception:
        return None


def reference_plan_bytes(spec, tp_src: int, dp_src: int, tp_tgt: int, samples: int, ctx: int) -> dict:
    """The reference's priced plans for the same switch (reported beside the executed
    bytes): per-rank received bytes of plan_weight_reshard / plan_kv_migration
    (tpshift/reshard.py:80-151, restated bit-exactly). The reference prices KV at the full hidden
    width per token (2 H bytes per layer); the executor moves the GQA heads (2 n_kv D)."""
    from paper_2605_23945_b200.reshard import ShardLayout, plan_kv_migration, plan_weight_reshard
    from paper_2605_23945_b200.workload import Sample
    H = spec.model.hidden_dim
    w = plan_weight_reshard(spec.model, ShardLayout(tp=tp_src, dim=H), ShardLayout(tp=tp_tgt, dim=H))
    live = [Sample(id=i, prompt_len=spec.prompt_len, target_response_len=spec.l_max,
                   generated_len=ctx - spec.prompt_len, intra_dp_group=i % dp_src) for i in range(samples)]
    kv = plan_kv_migration(live, spec.model, tp_src, dp_src, tp_tgt)
    return {"weights": w.total_per_rank_bytes, "kv": kv.total_per_rank_bytes}


def switch_microbench(args, hbm_peak):
    """BASELINE config 5 on one device: a real Switch Executor run TP1/DP2 -> TP2/DP1 of the
    bench model in a virtual 2-rank world (both ranks on this GPU, so every pull is an HBM
    copy: the bound is the HBM copy peak, read + write). 16 live samples at context 4096."""
    import dataclasses
    from paper_2605_23945_b200.cache_manager import World
    from paper_2605_23945_b200.profiler import switch_probe
    ns = argparse.Namespace(model=args.model, per_gpu_batch=8, l_max=args.l_max, prompt_len=args.prompt_len,
                            seed=args.seed)
    spec, geom = build_spec(ns, 2)
    spec = dataclasses.replace(spec, initial_tp=1, global_batch=16)
    r = switch_probe(spec, geom, World.virtual(2), 2, 16, 4096, copy_mode=1)
    gc.collect()
    torch.cuda.empty_cache()
    ref_plan = reference_plan_bytes(spec, 1, 2, 2, 16, 4096)
    return {"config": f"c5: {args.model}, virtual TP1/DP2 -> TP2/DP1 on one B200, 16 samples at ctx 4096, "
                      f"TMA bulk copy engine",
            "weights_bytes": r["weights_bytes"], "kv_bytes": r["kv_bytes"], "copy_bytes": r["copy_bytes"],
            "copy_kernel_ms": r["copy_kernel_ms"], "copy_gbps": r["copy_gbps"],
            "roofline": {"bound": "hbm", "achieved": 2 * r["copy_gbps"], "peak": hbm_peak, "unit": "GB/s",
                         "frac": 2 * r["copy_gbps"] / hbm_peak, "note": "read+write bytes of the copy kernels"},
            "switch_device_ms": r["switch_device_ms"], "release_to_resume_ms": r["release_to_resume_ms"],
            "max_gpu_peer_bytes": r["max_gpu_peer_bytes"], "max_gpu_local_bytes": r["max_gpu_local_bytes"],
            "host_switch_s": r["host_switch_s"], "host_plan_s": r["host_plan_s"],
            "host_capture_s": r["host_capture_s"], "reference_plan_bytes_per_rank": ref_plan,
            "note": "every rank on this GPU: a peer pull is an HBM copy; switch_device_ms runs from the first "
                    "rank's arrival at the opening barrier to the last rank's resume, host work included"}


def reference_arm(args):
    """The reference-side CPU path on the host cores (rank 0 only): the CPU oracle port of the
    decode step at full depth (the reference itself has no decode arithmetic),
    timed per step and composed over the stage's rounds, plus the reference's own decision
    layer (evaluate / run, restated bit-exact) timed single-threaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_23945_b200.engine import run as sim_run
    spec, geom = build_spec(args, max(1, args.gpus))
    threads = args.cpu_threads or os.cpu_count()
    # the stage's round profile (active batch per round) comes from the reference's own loop
    # on the analytic model: identical samples, lengths and block structure
    rep = sim_run(dataclasses.replace(spec, mode="static"))
    hist = active_histogram(rep)
    ctx = stage_mean_context(spec)
    cpu = CpuOracleSteps(geom, threads, ctx)
    for _ in range(args.warmup):  # warm-up passes: one B=1 step each (the full pass is ~30 s)
        cpu.orc.step([1], [ctx - 1], [0])
    vals = []
    for _ in range(args.steps):
        steps = cpu.measure()
        vals.append(cpu_stage_estimate(spec, steps, hist))
    value = float(np.mean(vals))
    sample = (f"CPU oracle (torch fp32 with bf16 rounding, {threads} threads) at full depth: decode steps at B="
              + ",".join(str(b) for b in steps["steps"]) + f", ctx {ctx}, and a 64-token prefill chunk, "
              f"composed over the stage's {sum(hist.values())} rounds at their active batch")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"c2-weak: {args.model}, {args.per_gpu_batch} samples/GPU, l_max {args.l_max}",
                   "model": args.model, "global_batch": spec.global_batch},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "measured_steps_s": {str(b): t for b, t in steps["steps"].items()},
                         "decision_layer": decision_layer_timing(args),
                         "switch": cpu_switch_baseline(args.model, threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
