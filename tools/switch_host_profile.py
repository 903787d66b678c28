"""Dev probe: cProfile of the host side of one Switch Executor run (config-5 point)."""
import argparse, cProfile, dataclasses, io, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.controller import assign_merged_groups
from paper_2605_23945_b200.coordinator import B200Backend
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.workload import BatchStatus, Sample

world, t0, t1, n, ctx = (int(x) for x in (sys.argv[1:] + ["2", "1", "2", "16", "4096"][len(sys.argv) - 1:])[:5])
ns = argparse.Namespace(model="qwen2.5-7b", per_gpu_batch=max(1, n // world), l_max=ctx, prompt_len=512, seed=4)
spec, geom = bench.build_spec(ns, world)
spec = dataclasses.replace(spec, initial_tp=t0, global_batch=n)
be = B200Backend(spec, geom, World.virtual(world), seed=0)
be.capture_all(every_layout=True)
be.prepare_switch_items()
for rep in range(2):
    be.reset(0)
    lay = be.layout
    samples = {g: [] for g in range(lay.dp)}
    prompt = torch.zeros(spec.prompt_len, dtype=torch.int32)
    for i in range(n):
        g = i % lay.dp
        slot = admit(be.group_ranks(g), i, prompt, max_ctx=be.max_len)
        be.slot_of[i] = slot
        samples[g].append(Sample(id=i, prompt_len=spec.prompt_len, target_response_len=spec.l_max,
                                 generated_len=ctx - spec.prompt_len, intra_dp_group=g))
    merged = assign_merged_groups([BatchStatus(0, g, tuple(v)) for g, v in samples.items()], t1, spec.cluster)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    be._execute_switch(t1, merged)
    pr.disable()
    torch.cuda.synchronize()
    t = be.switches[-1]
    print(f"rep {rep}: host_s {t.host_s*1e3:.2f} ms plan {t.host_plan_s*1e3:.2f} build {t.host_build_s*1e3:.2f}")
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25)
    print(s.getvalue()[:6000])
