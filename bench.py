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
  cpu_baseline  the CPU oracle (oracle/decoder_ref.py) on this host's cores,
             1 layer timed and extrapolated to the stage's round/batch profile

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
    ap.add_argument("--static-tps", default="1", help="N>1: also time the stage at these fixed TP degrees")
    ap.add_argument("--tp-list", default="", help="Algorithm 1 candidates (default: 1 and N, BASELINE config 2)")
    ap.add_argument("--initial-tp", type=int, default=1, help="starting TP degree (config 4 starts at TP2)")
    ap.add_argument("--cpu-threads", type=int, default=0)
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


def cpu_step_model(geom, threads: int, ctx: int = 2048):
    """Time the CPU oracle: one decoder layer at B in {1, 64} and the LM head; returns t(B) in s."""
    from oracle.decoder_ref import OracleDecoder
    torch.set_num_threads(threads)
    H, D, F = geom.hidden, geom.head_dim, geom.ffn
    geo = dict(num_layers=1, hidden=H, n_q=geom.n_q, n_kv=geom.n_kv, head_dim=D, ffn=F, vocab=256,
               qkv_bias=geom.qkv_bias, rope_theta=geom.rope_theta, rms_eps=geom.rms_eps)
    z = torch.zeros
    W = {(-1, "embed"): z(256, H), (-1, "ln_f"): torch.ones(H), (-1, "lm_head"): z(256, H),
         (0, "w_qkv"): z(geom.qkv_rows, H), (0, "b_qkv"): z(geom.qkv_rows), (0, "w_o"): z(H, geom.n_q * D),
         (0, "w_gu"): z(2 * F, H), (0, "w_d"): z(H, F), (0, "ln1"): torch.ones(H), (0, "ln2"): torch.ones(H)}
    lm = z(geom.vocab, H)
    times = {}
    for B in (1, 64):
        orc = OracleDecoder(geo, W, tp=1, round_bf16=True, max_len=ctx + 8)
        orc.step([1] * B, [ctx - 1] * B, list(range(B)))  # allocate caches, warm
        t0 = time.perf_counter()
        reps = 2
        for _ in range(reps):
            orc.step([1] * B, [ctx - 1] * B, list(range(B)))
        layer = (time.perf_counter() - t0) / reps
        x = torch.zeros(B, H)
        t0 = time.perf_counter()
        for _ in range(reps):
            _ = x @ lm.T
        head = (time.perf_counter() - t0) / reps
        times[B] = geom.num_layers * layer + head
    a = times[1]
    b = (times[64] - times[1]) / 63.0
    return (lambda B: a + b * (B - 1)), times


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import paper_2605_23945_b200 as pkg  # noqa: F401
    from paper_2605_23945_b200.cache_manager import World
    from paper_2605_23945_b200.coordinator import GlobalCoordinator
    from paper_2605_23945_b200.profiler import gemm_probe

    gpus = max(1, args.gpus)
    world = World.from_env() if gpus > 1 else World.virtual(1)
    rank = world.local_ranks[0]
    dev = world.devices[rank]
    spec, geom = build_spec(args, gpus)
    table = measured_table(args.model)
    t_setup = time.perf_counter()
    coord = GlobalCoordinator(spec, geom, world, seed=0, table=table)
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
    peak, peak_src = peaks()
    achieved = g_bytes / g_ms / 1e6
    switch = [s for nr in rep.node_reports for s in nr["switches"]]
    sw_gbps = [s.get("copy_gbps_per_gpu") for s in switch if s.get("copy_gbps_per_gpu")]
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
                      "seconds": s["breakdown"]["total"], "gbps_per_gpu": s.get("copy_gbps_per_gpu")}
                     for s in switch],
        "switch_gbps": (sum(sw_gbps) / len(sw_gbps)) if sw_gbps else None,
        "wall_s_per_step": float(np.mean(walls)),
        "setup_s": setup_s,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "kernel": "gemm_swapab_kernel (tcgen05)",
                     "peak_source": peak_src,
                     "per_bucket": {str(B): {"gbps": probes[B]["gbps"], "rounds": hist[B]} for B in sorted(hist)},
                     "rounds_at_other_tp": other_rounds},
        "clocks": clk.summary(),
    }
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
        line["roofline"]["traffic"] = tr["dram_bytes"]
        line["roofline"]["traffic_note"] = (f"ncu dram read+write of one launch ({tr['launch']}) vs its "
                                            f"{tr['algorithmic_bytes']} algorithmic bytes; profiles/r1/ncu_traffic.json")
    if gpus > 1 and args.static_tps:
        # the north-star comparison: the same stage at a fixed TP (no switching), same engine
        line["fixed_tp"] = {}
        for tp in (int(x) for x in args.static_tps.split(",")):
            if gpus % tp:
                continue
            ex = coord = None
            gc.collect()  # executors / runners / comms form reference cycles
            torch.cuda.empty_cache()
            sspec = dataclasses.replace(spec, mode="static", initial_tp=tp)
            coord = GlobalCoordinator(sspec, geom, world, seed=0, table=table)
            coord.run()
            srep, _ = coord.run()
            line["fixed_tp"][str(tp)] = srep.generation_time
    if rank == 0 and gpus == 1 and not args.no_switch:
        line["switch_microbench"] = switch_microbench(args, peak)
    if rank == 0 and gpus == 1 and not args.no_cpu:
        threads = args.cpu_threads or os.cpu_count()
        step_t, raw = cpu_step_model(geom, threads)
        est = (args.prompt_len - 1) * step_t(spec.global_batch)
        for B, n in hist.items():
            est += n * step_t(B)
        line["cpu_baseline"] = {"value": est, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"CPU oracle: 1 decoder layer + LM head timed at B=1 "
                                          f"({raw[1]*1e3:.0f} ms/step x28 layers) and B=64 "
                                          f"({raw[64]*1e3:.0f} ms/step), ctx 2048, extrapolated over the "
                                          f"stage's {sum(hist.values())} rounds and prefill"}
    if rank == 0:
        print(json.dumps(line), flush=True)


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
    None (the analytic b200.cfg calibration) when the model has not been profiled."""
    from paper_2605_23945_b200.latency import load_table
    path = os.path.join(HERE, "paper_2605_23945_b200", "presets", f"b200_{model}_profile.csv")
    return load_table(path) if os.path.exists(path) else None


def traffic_record():
    try:
        with open(os.path.join(HERE, "profiles", "r1", "ncu_traffic.json")) as fh:
            return json.load(fh)["gemm_swapab_kernel"]
    except Exception:
        return None


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
    return {"config": f"c5: {args.model}, virtual TP1/DP2 -> TP2/DP1 on one B200, 16 samples at ctx 4096, "
                      f"TMA bulk copy engine",
            "weights_bytes": r["weights_bytes"], "kv_bytes": r["kv_bytes"], "copy_bytes": r["copy_bytes"],
            "copy_kernel_ms": r["copy_kernel_ms"], "copy_gbps": r["copy_gbps"],
            "roofline": {"bound": "hbm", "achieved": 2 * r["copy_gbps"], "peak": hbm_peak, "unit": "GB/s",
                         "frac": 2 * r["copy_gbps"] / hbm_peak, "note": "read+write bytes of the copy kernels"},
            "switch_device_ms": r["switch_device_ms"], "host_plan_s": r["host_plan_s"],
            "host_capture_s": r["host_capture_s"]}


def reference_arm(args):
    """The reference-side CPU path: the oracle port on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_23945_b200.engine import run as sim_run
    from paper_2605_23945_b200.models import geometry
    spec, geom = build_spec(args, max(1, args.gpus))
    threads = args.cpu_threads or os.cpu_count()
    # the stage's round profile (batch per round) comes from the reference's own loop on the
    # analytic model: identical samples, lengths and block structure
    import dataclasses
    rep = sim_run(dataclasses.replace(spec, mode="static"))
    hist = {}
    for nr in rep.node_reports:
        for ev in nr["events"]:
            if ev["type"] == "step-block":
                lo, hi = (int(x) for x in ev["detail"].split("=")[1].split(".."))
                hist[ev["active"]] = hist.get(ev["active"], 0) + (hi - lo)
    vals = []
    for _ in range(args.warmup + args.steps):
        step_t, raw = cpu_step_model(geom, threads)
        est = (args.prompt_len - 1) * step_t(spec.global_batch)
        for B, n in hist.items():
            est += n * step_t(B)
        vals.append(est)
    value = float(np.mean(vals[args.warmup:]))
    sample = (f"CPU oracle (torch fp32, {threads} threads): 1 decoder layer + LM head at B=1 and B=64, ctx "
              f"2048, extrapolated to {geom.num_layers} layers and the stage's {sum(hist.values())} rounds")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"c2-weak: {args.model}, {args.per_gpu_batch} samples, l_max {args.l_max}",
                   "model": args.model, "global_batch": spec.global_batch},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
