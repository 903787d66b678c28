"""Worker for test_gpu_multiprocess.py: one adaptive stage, one process per rank (torchrun).

Run with TPS_SHARE_DEVICE=1 on a 1-GPU box: every rank's process uses cuda:0, so
the peer pointers are real CUDA-IPC mappings between processes, the TP allreduce
and the switch barriers spin on counters written by another process, and the
switch pulls go through IPC-opened peer memory -- the multi-GPU path, minus
NVLink. Each rank saves the sample ids it retired as TP lead and their tokens.
"""

import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    out_dir = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else "tiny"
    method = sys.argv[3] if len(sys.argv) > 3 else ""
    from paper_2605_23945_b200.cache_manager import World
    from paper_2605_23945_b200.coordinator import GlobalCoordinator
    from paper_2605_23945_b200.models import geometry
    from test_gpu_coordinator import tiny_spec

    world = World.from_env()
    geom = geometry(name)
    spec = tiny_spec(geom, gpus=world.gpus)
    coord = GlobalCoordinator(spec, geom, world, seed=7, state_method=method or None)
    report, meas = coord.run()
    rank = world.local_ranks[0]
    ids = list(coord.backend.retired_here)
    torch.save({"ids": ids, "tokens": coord.outputs()[ids].clone(),
                "switches": [(s["from_tp"], s["to_tp"], s["round"]) for nr in report.node_reports
                             for s in nr["switches"]],
                "tokens_generated": report.tokens_generated},
               os.path.join(out_dir, f"mp_rank{rank}.pt"))
    world.barrier()
    print(f"rank {rank}: retired {len(ids)} samples, switches "
          f"{[(s['from_tp'], s['to_tp']) for nr in report.node_reports for s in nr['switches']]}", flush=True)


if __name__ == "__main__":
    main()
