"""Switch Executor microbench (BASELINE config 5) on one device: virtual-world switches, copy GB/s."""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.profiler import switch_probe

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen2.5-7b")
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--pairs", default="1:2")
ap.add_argument("--samples", default="16")
ap.add_argument("--ctx", default="4096")
ap.add_argument("--modes", default="0,1")
a = ap.parse_args()
for pair in a.pairs.split(","):
    t0, t1 = (int(x) for x in pair.split(":"))
    for n in (int(x) for x in a.samples.split(",")):
        for ctx in (int(x) for x in a.ctx.split(",")):
            ns = argparse.Namespace(model=a.model, per_gpu_batch=max(1, n // a.world), l_max=max(ctx, 1024),
                                    prompt_len=512, seed=4)
            spec, geom = bench.build_spec(ns, a.world)
            spec = dataclasses.replace(spec, initial_tp=t0, global_batch=n)
            for mode in (int(x) for x in a.modes.split(",")):
                r = switch_probe(spec, geom, World.virtual(a.world), t1, n, ctx, copy_mode=mode)
                r.update(model=a.model, world=a.world, tp=f"{t0}->{t1}", samples=n, ctx=ctx, mode=mode)
                print(json.dumps(r), flush=True)
                torch.cuda.empty_cache()
