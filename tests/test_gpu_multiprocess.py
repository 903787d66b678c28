"""The one-process-per-GPU path (CUDA IPC peer tables, cross-process counters) on one B200.

torchrun starts `world` worker processes that all use cuda:0 (TPS_SHARE_DEVICE=1):
every peer pointer is a cudaIpcOpenMemHandle mapping of another process's
buffer, exactly as on an 8-GPU node, and every wait spins on a counter another
process's kernel releases. The stage runs Algorithm 1 with live switches; the
tokens every process retires must equal, bit for bit, the tokens of the same
stage in a single-process virtual world (same kernels, same fixed reduction
order), and must be complete (every sample retired exactly once).
"""

import os
import subprocess
import sys

import pytest
import torch

from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.coordinator import GlobalCoordinator
from paper_2605_23945_b200.models import geometry

from test_gpu_coordinator import tiny_spec

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _launch(tmp_path, world: int, name: str, method: str = "") -> list[dict]:
    env = dict(os.environ, TPS_SHARE_DEVICE="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "tests", "mp_stage_worker.py"), str(tmp_path), name, method]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    if res.returncode != 0:
        keep = [ln for ln in (res.stdout + res.stderr).splitlines() if "tps watchdog" not in ln]
        raise AssertionError("\n".join(keep[:80]) + "\n...\n" + "\n".join(keep[-40:]))
    return [torch.load(tmp_path / f"mp_rank{r}.pt") for r in range(world)]


@pytest.mark.parametrize("name,method", [("tiny", ""), ("mini-qwen", ""), ("tiny", "recompute")])
def test_ipc_processes_match_virtual_world(tmp_path, name, method):
    world = 4
    parts = _launch(tmp_path, world, name, method)
    geom = geometry(name)
    spec = tiny_spec(geom, gpus=world)
    coord = GlobalCoordinator(spec, geom, World.virtual(world), seed=7, state_method=method or None)
    report, _ = coord.run()
    ref = coord.outputs()
    sw = [(s["from_tp"], s["to_tp"], s["round"]) for nr in report.node_reports for s in nr["switches"]]
    assert sw, "controller never switched"
    seen = []
    for p in parts:
        assert p["switches"] == sw  # SPMD: every process reached the same decisions
        assert p["tokens_generated"] == report.tokens_generated
        seen += p["ids"]
        assert torch.equal(p["tokens"], ref[p["ids"]])
    assert sorted(seen) == list(range(spec.global_batch))
