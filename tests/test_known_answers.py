"""Known-answer constants of the reference test-suite (pkg/tests/*), restated against this package.

Each constant is cited to the reference test that pins it.
"""

import math

import numpy as np
import pytest

from paper_2605_23945_b200.cluster import ClusterSpec, ModelSpec, ParallelConfig, candidate_configs
from paper_2605_23945_b200.config import build_scenario, load_config
from paper_2605_23945_b200.controller import ControllerParams, compute_merged_bs
from paper_2605_23945_b200.engine import build_hardware_model, build_profile, reference_switch_costs, run
from paper_2605_23945_b200.errors import ConfigError, PlanVerificationError, ProfileLookupError, ScenarioError
from paper_2605_23945_b200.latency import (OracleLatencyModel, fit_predictor, oracle_decode_latency,
                                          oracle_prefill_latency, profile_batches, profile_lengths)
from paper_2605_23945_b200.reshard import ShardLayout, plan_kv_migration, plan_weight_reshard, verify_plan
from paper_2605_23945_b200.switchcost import (MIGRATE, CommGroupPool, GraphCaptureCalibration,
                                              comm_group_cost, graph_recapture_cost, kv_migration_time,
                                              kv_send_bytes_per_rank, naive_switch_cost, total_switch_cost,
                                              weight_reshard_time)
from paper_2605_23945_b200.workload import Sample

KV_BYTES_PER_RANK_PROBE = 28991029248          # pkg/tests/test_switchcost.py:16
KV_MOVE_S_PROBE = 2.3600642500814066           # pkg/tests/test_switchcost.py:17
WEIGHT_RESHARD_S_2_TO_8 = 0.9942863275805927   # pkg/tests/test_switchcost.py:18
DECODE_ANCHORS = {(2, 1, 4096): 0.015370032885333606, (8, 1, 4096): 0.009640032221333401}  # test_latency.py:14-17
PREFILL_9x12288_TP8 = 19.010039375872005       # pkg/tests/test_latency.py:18


@pytest.fixture(scope="module")
def a40():
    return load_config("paper_a40")


@pytest.fixture(scope="module")
def hw(a40):
    return build_hardware_model(build_scenario(a40))


def probe(n=9, ctx=12288, prompt=512):
    return [Sample(id=i, prompt_len=prompt, target_response_len=ctx - prompt, generated_len=ctx - prompt)
            for i in range(n)]


def test_kv_volume_probe(a40):
    assert kv_send_bytes_per_rank(probe(), a40.model, 2) == KV_BYTES_PER_RANK_PROBE
    assert kv_migration_time(KV_BYTES_PER_RANK_PROBE, a40.cluster) == pytest.approx(KV_MOVE_S_PROBE, rel=1e-12)
    s = probe()
    s[0].status = "finished"
    assert kv_send_bytes_per_rank(s, a40.model, 2) == KV_BYTES_PER_RANK_PROBE * 8 // 9


def test_weight_reshard_probe(a40):
    assert weight_reshard_time(a40.model, 8, a40.cluster) == pytest.approx(WEIGHT_RESHARD_S_2_TO_8, rel=1e-12)
    assert weight_reshard_time(a40.model, 1, a40.cluster) == 0.0


def test_decode_and_prefill_anchors(hw):
    for (tp, b, agg), want in DECODE_ANCHORS.items():
        assert oracle_decode_latency(hw, tp, b, float(agg)) == pytest.approx(want, rel=1e-12)
    assert oracle_prefill_latency(hw, 8, 9, 12288.0) == pytest.approx(PREFILL_9x12288_TP8, rel=1e-12)
    t2 = oracle_decode_latency(hw, 2, 128, 65536.0)
    t8 = oracle_decode_latency(hw, 8, 128, 65536.0)
    assert t8 / t2 == pytest.approx(1.2646, abs=2e-3)  # test_latency.py:27-31


def test_total_switch_probe_and_reference_breakdown(a40, hw):
    pool = CommGroupPool.fresh(a40.switch.comm_init_cost, warm=((8, 1),))
    bd = total_switch_cost(OracleLatencyModel(hw), pool, a40.switch, probe(), 2, 8, a40.model, a40.cluster)
    assert bd.state_method == MIGRATE
    assert bd.t_graph_recapture == pytest.approx(0.73)
    assert bd.total == pytest.approx(KV_MOVE_S_PROBE + WEIGHT_RESHARD_S_2_TO_8 + 0.73 + 1.40)
    cold = CommGroupPool.fresh(a40.switch.comm_init_cost)
    bd2 = total_switch_cost(OracleLatencyModel(hw), cold, a40.switch, probe(), 2, 8, a40.model, a40.cluster)
    assert bd2.t_comm_group_init == pytest.approx(0.30) and (8, 1) not in cold.initialized
    ref = reference_switch_costs(build_scenario(a40), build_profile(build_scenario(a40)))
    assert ref["incremental"]["total"] == pytest.approx(5.484, abs=2e-3)  # pkg/README.md:112-116
    assert naive_switch_cost(a40.switch.naive).total == pytest.approx(58.98)


def test_graph_bucket_rule():
    calib = GraphCaptureCalibration()
    for merged, n in {1: 1, 2: 2, 3: 3, 4: 3, 8: 4, 9: 5, 16: 5, 17: 6, 32: 6}.items():
        assert graph_recapture_cost(calib, merged) == pytest.approx(0.146 * n)
    assert graph_recapture_cost(calib, 33) == 0.0
    with pytest.raises(ConfigError):
        graph_recapture_cost(calib, 0)


def test_pool_grows_only():
    pool = CommGroupPool.fresh(0.3, warm=((2, 4),))
    c, same = comm_group_cost(pool, 2, 4)
    assert c == 0.0 and same is pool
    c, grown = comm_group_cost(pool, 8, 1)
    assert c == 0.3 and (8, 1) in grown.initialized and (8, 1) not in pool.initialized


def test_kv_plan_probe(a40):
    samples = [Sample(id=i, prompt_len=512, target_response_len=11776, generated_len=11776, intra_dp_group=i % 4)
               for i in range(9)]
    plan = plan_kv_migration(samples, a40.model, 2, 4, 8)
    assert plan.peak_working_bytes == 1811939328  # pkg/tests/test_reshard.py:67-77
    assert verify_plan(plan, ShardLayout(tp=8, dim=4096)) == []


def test_all_transitions_verify_clean():
    model = ModelSpec(name="probe", num_layers=3, hidden_dim=64, bytes_per_elem=2, layer_param_bytes=8192)
    for s in (1, 2, 4, 8):
        for t in (1, 2, 4, 8):
            assert verify_plan(plan_weight_reshard(model, ShardLayout(s, 64), ShardLayout(t, 64)),
                               ShardLayout(t, 64)) == []


def test_profile_grid_shape():
    assert profile_batches() == [1, 2, 3, 6, 12, 22, 40, 75, 138, 256]
    ls = profile_lengths()
    assert [l for l in ls if l <= 512] == [8, 11, 16, 23, 32, 45, 64, 91, 128, 181, 256, 362, 512]
    assert ls[-1] == 131072


def test_predictor_exact_on_grid_and_rejects_unknown_tp(a40):
    spec = build_scenario(a40)
    table = build_profile(spec)
    pred = fit_predictor(table)
    for p in table.points[::37]:
        assert pred.predict_decode_latency(p.tp, p.batch, p.batch * p.ctx_len) == pytest.approx(
            p.decode_latency, rel=1e-12)
    with pytest.raises(ProfileLookupError):
        pred.predict_decode_latency(3, 1, 100.0)


def test_compute_merged_bs_table():
    cl = ClusterSpec(num_nodes=1, gpus_per_node=8, intra_bw_unidir=1e9, kv_tokens_per_gpu=65536, hbm_bw=1e12,
                     peak_flops=1e14, per_layer_tp_comm_base=1e-5)
    assert compute_merged_bs([3, 3, 2, 2], 4, cl) == [5, 5]
    assert compute_merged_bs([3, 3, 2, 2], 1, cl) == [2, 2, 1, 1, 1, 1, 1, 1]
    assert compute_merged_bs([9], 2, cl) == [3, 2, 2, 2]


def test_default_scenario_reproduces_readme(a40):
    rep = run(build_scenario(a40))
    assert rep.generation_time == pytest.approx(227.8, abs=0.05)  # pkg/README.md:17-22


def test_validation_errors(a40):
    with pytest.raises(ConfigError):
        ControllerParams(tp_list=(4, 2))
    with pytest.raises(ConfigError):
        ShardLayout(tp=3, dim=64)
    with pytest.raises(ConfigError):
        ParallelConfig(tp=3, dp_intra=1, dp_inter=1)
    with pytest.raises(ScenarioError):
        build_scenario(a40, mode="bogus")
    assert [c.tp for c in candidate_configs(a40.cluster)] == [1, 2, 4, 8]
    assert issubclass(PlanVerificationError, Exception)
