"""The bench's own stages through the UNMODIFIED reference, CPU only (container).

bench.py's workloads -- BASELINE configs 2-4 (Qwen2.5-7B, Llama-3-8B, Qwen2.5-32B shapes, 64
samples per GPU, long-tail lengths scaled to the cap, Algorithm 1 over the TP degrees dividing N)
on the B200-measured profile tables, at N = 1, 2, 4, 8, adaptive and fixed-TP -- are run by the
reference simulator itself (tpshift.run, /root/reference/pkg/src, tpshift/engine.py:461-515) and
by this package's restated loop (engine.run); the SimReport JSON must be byte-identical. This
pins the decision layer on exactly the inputs the benchmark feeds it (the golden-vector tests pin
it on the reference's own presets). The values are converted with bench.to_reference, the same
conversion bench.py's `cpu_baseline.decision_layer.reference_impl` timing uses.
"""

import argparse
import dataclasses
import sys

import pytest

import bench
from paper_2605_23945_b200.engine import run as ours

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def T():
    sys.path.insert(0, "/root/reference/pkg/src")
    import tpshift
    return tpshift


CASES = [("qwen2.5-7b", 8192, 1), ("llama3-8b", 16384, 1), ("qwen2.5-32b", 16384, 2)]


@pytest.mark.parametrize("model,l_max,init_tp", CASES)
@pytest.mark.parametrize("gpus", [1, 2, 4, 8])
def test_bench_stage_identical_to_reference(T, model, l_max, init_tp, gpus):
    if gpus % init_tp:
        pytest.skip("initial TP does not divide N")
    ns = argparse.Namespace(model=model, per_gpu_batch=64 if model != "qwen2.5-32b" else 16, l_max=l_max,
                            prompt_len=512, seed=4, tp_list="1,2,4,8", initial_tp=init_tp)
    spec, _ = bench.build_spec(ns, gpus)
    table = bench.measured_table(model)
    assert table is not None
    for mode in ("adaptive", "static"):
        s = spec if mode == "adaptive" else dataclasses.replace(spec, mode="static")
        mine = ours(s, table).to_json()
        ref = T.run(bench.to_reference(T, s), bench.to_reference(T, table)).to_json()
        assert mine == ref, (model, gpus, mode)
