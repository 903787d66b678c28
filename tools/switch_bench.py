"""Switch Executor microbench (BASELINE config 5) on one device: virtual-world switches.

Sweep: model x active samples x context x (tp -> tp') at world sizes 2/4/8 (every rank of the
virtual world on this GPU, so a "peer" pull is an HBM copy: read + write at the HBM copy
peak). DP replicas of one TP rank share their weight arena (--alias, default on: replicas hold
identical canonical shards) so 8-rank worlds of 7B/8B/32B fit one device; points whose pools
still do not fit are reported as skipped. One JSON line per point.

python tools/switch_bench.py [--models qwen2.5-7b,llama3-8b,qwen2.5-32b] [--worlds 2,4,8]
       [--samples 1,4,16,64] [--ctx 4096,8192,16384] [--pairs all|1:2,...] [--mode 1]
"""
import argparse, dataclasses, gc, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.kvcache import pages_for
from paper_2605_23945_b200.models import geometry, rank_shard
from paper_2605_23945_b200.profiler import switch_probe
from paper_2605_23945_b200.shards import arena_layout

ap = argparse.ArgumentParser()
ap.add_argument("--models", default="qwen2.5-7b")
ap.add_argument("--worlds", default="2")
ap.add_argument("--pairs", default="all")
ap.add_argument("--samples", default="16")
ap.add_argument("--ctx", default="4096")
ap.add_argument("--mode", type=int, default=1)
ap.add_argument("--no-alias", action="store_true")
ap.add_argument("--budget-gb", type=float, default=165.0)
a = ap.parse_args()


def est_bytes(geom, world, tp, n, max_len, alias):
    """HBM of one layout in a virtual world: weight shards (aliased replicas) + KV pools."""
    dp = world // tp
    slots = max(1, -(-n // dp))
    tot = 0
    for r in range(world):
        sh = rank_shard(geom, tp, r % tp)
        if not alias or r < tp:
            tot += arena_layout(geom, sh).total_bytes
        tot += geom.num_layers * 2 * slots * pages_for(max_len) * sh.n_kv * 64 * geom.head_dim * 2
    return tot


def ok_tp(geom, tp):
    try:
        geom.check_tp(tp)
        return True
    except Exception:
        return False


for model in a.models.split(","):
    geom = geometry(model)
    for world in (int(x) for x in a.worlds.split(",")):
        tps = [t for t in (1, 2, 4, 8) if world % t == 0 and t <= world and ok_tp(geom, t)]
        pairs = [(x, y) for x in tps for y in tps if x != y] if a.pairs == "all" else \
            [tuple(int(v) for v in p.split(":")) for p in a.pairs.split(",")]
        for t0, t1 in pairs:
            if world % t0 or world % t1:
                continue
            for n in (int(x) for x in a.samples.split(",")):
                for ctx in (int(x) for x in a.ctx.split(",")):
                    pt = dict(model=model, world=world, tp=f"{t0}->{t1}", samples=n, ctx=ctx, mode=a.mode)
                    l_max = max(ctx, 1024)
                    need = est_bytes(geom, world, t0, n, 512 + l_max, not a.no_alias) + \
                        est_bytes(geom, world, t1, n, 512 + l_max, not a.no_alias)
                    if need > a.budget_gb * 2 ** 30:
                        print(json.dumps(dict(pt, skipped=f"needs ~{need / 2 ** 30:.0f} GB on one device")), flush=True)
                        continue
                    ns = argparse.Namespace(model=model, per_gpu_batch=max(1, -(-n // world)), l_max=l_max,
                                            prompt_len=512, seed=4, tp_list=f"{min(t0, t1)},{max(t0, t1)}",
                                            initial_tp=t0)
                    spec, _ = bench.build_spec(ns, world)
                    spec = dataclasses.replace(spec, initial_tp=t0, global_batch=n)
                    try:
                        r = switch_probe(spec, geom, World.virtual(world), t1, n, ctx, copy_mode=a.mode,
                                         alias_replicas=not a.no_alias, use_graphs=False)
                    except torch.cuda.OutOfMemoryError as e:
                        r = {"skipped": "CUDA OOM"}
                    r.update(pt)
                    if "copy_kernel_ms" in r:
                        r["device_over_copy"] = r["switch_device_ms"] / max(r["copy_kernel_ms"], 1e-9)
                    print(json.dumps(r), flush=True)
                    gc.collect()
                    torch.cuda.empty_cache()
