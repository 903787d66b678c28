"""Dev probe: one rank of a TP-k group alone on the GPU (peer tables loop back to itself).

Every allreduce push lands in the rank's own receive area and its signal list holds
its own counter tp times, so waits complete; numerics are meaningless but the step
runs exactly the kernels (and sizes) a real TP-k rank runs, minus the NVLink hop.
"""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.executor import GroupRunner
from paper_2605_23945_b200.group import admit, build_rank
from paper_2605_23945_b200.models import geometry


def solo(geom, tp, maxb, ctx, rank=0):
    from paper_2605_23945_b200.profiler import loopback_rank
    from paper_2605_23945_b200.kvcache import pages_for
    return loopback_rank(geom, tp, maxb, maxb, ctx + 256, maxb * pages_for(ctx + 256))


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
    tps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
    batches = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 16, 64]
    ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
    variants = sys.argv[5].split(";") if len(sys.argv) > 5 else [""]
    geom = geometry(name)
    for tp in tps:
        r, runner = solo(geom, tp, max(batches), ctx)
        slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(max(batches))]
        wb = r.weights.nbytes - (geom.vocab // tp) * geom.hidden * 2 * 0  # shard bytes (embedding replicated)
        for B in batches:
            bk = r.executor.bucket(B)
            runner.set_rows(bk, slots[:B])
            for v in variants:
                toks = [x for x in v.split(",") if x]
                r.executor.fuse_silu_min_units = 0 if "+silu_fused" in toks else (10 ** 9 if "+silu_unfused" in toks
                                                                                  else 120)
                r.executor.skip = frozenset(x for x in toks if not x.startswith("+"))
                r.slots.pos[:] = ctx
                runner.graphs.pop(bk, None)
                runner.step(bk, 1)
                runner.capture(bk)
                runner.step(bk, 3)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n = 20
                e0.record(); runner.step(bk, n); e1.record(); torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / n
                print(f"{name} solo tp={tp} B={B:3d} ctx={ctx} [{v or 'default'}] step {ms:.3f} ms "
                      f"kernels/step {runner.kernels_per_step(bk)}", flush=True)
        del r, runner
        torch.cuda.empty_cache()
