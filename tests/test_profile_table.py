"""The B200 Offline Profiler's committed table (presets/b200_qwen2.5-7b_profile.csv).

It is written by tools/profile_b200.py on a B200 in the reference's CSV schema
(tpshift/latency.py:376-391) and drives Algorithm 1 in bench.py at N > 1. These CPU
tests pin its schema and that the reference's loop runs on it, both as the planner's
predictor and as the replayed ground truth (engine.TableBackend)."""

import argparse
import dataclasses
import os

import pytest

from paper_2605_23945_b200.engine import TableBackend, run
from paper_2605_23945_b200.latency import fit_predictor, load_table, profile_batches
from paper_2605_23945_b200.workload import sample_response_lengths

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLE = os.path.join(ROOT, "paper_2605_23945_b200", "presets", "b200_qwen2.5-7b_profile.csv")


@pytest.fixture(scope="module")
def table():
    return load_table(TABLE)


def test_schema_and_coverage(table):
    assert table.tps == (1, 2, 4, 8)
    assert set(table.grid_batches) == set(profile_batches())
    assert table.token_cap == 1 << 20
    for p in table.points:
        assert p.batch * p.ctx_len <= table.token_cap
        assert 0 < p.decode_latency < 1.0 and p.prefill_latency > 0


def test_measured_tp_scaling_at_the_tail(table):
    """Tail decode (one sample) gets faster with TP on the measured B200 engine."""
    pred = fit_predictor(table)
    t = [pred.predict_decode_latency(tp, 1, 2048) for tp in (1, 2, 4, 8)]
    assert t[0] > t[1] > t[2] > t[3]


def test_reference_loop_replays_the_table():
    import bench
    tab = load_table(TABLE)
    ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=8, l_max=1024, prompt_len=128, seed=4)
    spec, _ = bench.build_spec(ns, 2)
    for s in (spec, dataclasses.replace(spec, mode="static")):
        rep = run(s, tab, TableBackend(s, tab))
        want = sum(min(t, s.l_max) for t in sample_response_lengths(s.distribution, s.global_batch, s.seed))
        assert rep.tokens_generated == want
        assert rep.generation_time > 0


def test_bench_stage_roofline_units():
    """bench.stage_roofline: the decode HBM floor of config 2's stage (SURVEY §8(d) units:
    all weight shards + every live sample's K/V per round) at the measured copy peak."""
    import argparse
    import bench
    ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=64, l_max=8192, prompt_len=512, seed=4, tp_list="",
                            initial_tp=1)
    spec, geom = bench.build_spec(ns, 1)
    r = bench.stage_roofline(spec, geom, decode_s=12.0, peak_gbps=6547.2)
    w = geom.num_layers * geom.layer_param_bytes + geom.vocab * geom.hidden * 2
    assert abs(w - 14.14e9) < 0.01e9                     # 14.14 GB at TP1
    assert r["rounds"] == 3104 and r["bytes"] > r["rounds"] * w
    assert abs(r["decode_floor_s"] - r["bytes"] / 6547.2e9) < 1e-9
    assert 0.6 < r["frac"] < 0.8


def test_bench_cpu_stage_estimate_composes_measured_steps():
    """cpu_baseline: the stage = every round at its active batch (piecewise-linear between the
    measured full-depth step times) + the prompts' prefill at the 64-token chunk rate."""
    import argparse
    import bench
    ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=64, l_max=8192, prompt_len=512, seed=4, tp_list="",
                            initial_tp=1)
    spec, _ = bench.build_spec(ns, 1)
    steps = {"steps": {1: 1.0, 8: 2.0, 64: 9.0}, "prefill64_s": 0.5}
    hist = {1: 10, 4: 3, 64: 2, 36: 1}
    got = bench.cpu_stage_estimate(spec, steps, hist)
    dec = 10 * 1.0 + 3 * (1.0 + 3 / 7) + 2 * 9.0 + 1 * (2.0 + 7.0 * 28 / 56)
    assert abs(got - (dec + 64 * 8 * 0.5)) < 1e-9
    rep = run(dataclasses.replace(spec, mode="static"))
    h = bench.active_histogram(rep)
    assert sum(h.values()) == 3104 and max(h) == 64
    assert 512 < bench.stage_mean_context(spec) < 8704


def test_switch_rate_is_max_gpu_peer_bytes_over_release_to_resume():
    """RecordedBackend's switch record: per GPU, bytes pulled from peers over that
    GPU's barrier-release -> resume window; the rate is the max over GPUs; local bytes apart."""
    from paper_2605_23945_b200.coordinator import RecordedBackend
    sw = {"ranks": {0: [1.0, 1.1, 1.2, 1.3, 1.4], 1: [1.05, 1.1, 1.25, 1.32, 1.5]},
          "per_rank": {0: {"nvlink": 30e9, "local": 5e9}, 1: {"nvlink": 20e9, "local": 1e9}},
          "nvlink_bytes": 50e9, "local_bytes": 6e9, "kv_bytes": 1e9, "weight_bytes": 55e9,
          "host_plan_s": 0.001, "host_capture_s": 0.0, "host_build_s": 0.0, "host_s": 0.002,
          "state_method": "migrate"}
    rb = RecordedBackend([{"groups": {}, "switches": [sw]}])
    rb.nswitch = 1
    rec = rb.switch_record_extra(None)
    assert abs(rec["release_to_resume_s"] - 0.4) < 1e-12
    assert rec["max_gpu_peer_bytes"] == 30e9 and rec["max_gpu_local_bytes"] == 5e9
    assert abs(rec["peer_gbps_per_gpu"] - max(30 / 0.3, 20 / 0.4)) < 1e-9


def test_monotone_table_is_monotone_and_close_to_the_measurement(table):
    from paper_2605_23945_b200.profiler import monotone_table
    sm = monotone_table(table)
    raw = {(p.tp, p.batch, p.ctx_len): p for p in table.points}
    fit = {(p.tp, p.batch, p.ctx_len): p for p in sm.points}
    assert raw.keys() == fit.keys() and sm.token_cap == table.token_cap
    for k, p in fit.items():
        assert abs(p.decode_latency - raw[k].decode_latency) <= 0.03 * raw[k].decode_latency
        assert p.prefill_latency == raw[k].prefill_latency
    for axis in (2, 1):
        groups = {}
        for k in fit:
            groups.setdefault((k[0], k[1]) if axis == 2 else (k[0], k[2]), []).append(k)
        for ks in groups.values():
            ys = [fit[k].decode_latency for k in sorted(ks, key=lambda k: k[axis])]
            assert all(b >= a - 1e-15 for a, b in zip(ys, ys[1:]))


def test_table_backend_switch_bytes_match_the_executed_plans():
    """switch_bytes_per_gpu (what TableBackend prices) = the weight pull plans' bytes + the KV
    chunk plan's bytes + history rows, per target rank, split into peer and local."""
    from paper_2605_23945_b200.models import geometry
    from paper_2605_23945_b200.switch_executor import (KVSource, KVTarget, Layout, cached_weight_pulls,
                                                       nvlink_bytes, plan_kv_pulls, switch_bytes_per_gpu)
    from paper_2605_23945_b200.workload import Sample
    geom = geometry("mini-qwen")
    old, new = Layout(2, 8), Layout(4, 8)
    samples = [Sample(id=i, prompt_len=8, target_response_len=100, generated_len=20 + 37 * i, intra_dp_group=i % 4)
               for i in range(6)]
    merged = [[s for s in samples if s.id % 2 == g] for g in range(2)]
    got = switch_bytes_per_gpu(geom, old, new, merged, lambda s: s.intra_dp_group, lambda s: s.context_len - 1)
    for r in range(8):
        nv, loc = nvlink_bytes(cached_weight_pulls(geom, old, new, r), r)
        mine = merged[new.group_of(r)]
        src = [KVSource(old_group=s.intra_dp_group, slot=0, pages=tuple(range(40))) for s in mine]
        tgt = [KVTarget(slot=0, pages=tuple(range(40))) for s in mine]
        kp = plan_kv_pulls(geom, old, new, r, src, tgt, [s.context_len - 1 for s in mine], 64, 64)
        a, b = nvlink_bytes(kp, r)
        h_nv = sum(4 * s.context_len for s in mine if r not in old.ranks_of_group(s.intra_dp_group))
        h_loc = sum(4 * s.context_len for s in mine if r in old.ranks_of_group(s.intra_dp_group))
        assert got[r] == (nv + a + h_nv, loc + b + h_loc), r


def test_bench_decision_layer_timing_runs_the_reference_path():
    """cpu_baseline.decision_layer: Algorithm 1 at B=512 (config 2 on 8 GPUs) and a whole
    simulated stage, timed single-threaded."""
    import argparse
    import bench
    d = bench.decision_layer_timing(argparse.Namespace(model="qwen2.5-7b", l_max=8192, prompt_len=512, seed=4))
    assert d["evaluate_live_samples"] > 400 and d["evaluate_ms"] > 0 and d["run_stage_s"] > 0


def test_table_backend_falls_back_to_the_quote_without_a_geometry():
    """A reference preset's model (no executable geometry) is priced by the planner's quote."""
    from paper_2605_23945_b200.config import build_scenario, load_config
    from paper_2605_23945_b200.engine import build_profile
    spec = build_scenario(load_config("paper_a40"), l_max=12288, seed=3)
    tab = build_profile(spec)
    rep = run(spec, tab, TableBackend(spec, tab))
    sw = [s for nr in rep.node_reports for s in nr["switches"]]
    assert sw and all(abs(s["breakdown"]["total"] - s["quoted_total"]) < 1e-12 for s in sw)
