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
