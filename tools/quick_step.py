"""Dev probe: graph-replayed decode-step time and per-kernel times for a geometry at TP1."""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import build_group, admit
from paper_2605_23945_b200.models import geometry

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
batches = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16, 64]
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
geom = geometry(name)
maxb = max(batches)
t0 = time.time()
ranks, runner = build_group(geom, 1, max_batch=maxb, num_slots=maxb, max_len=ctx + 256, seed=0)
torch.cuda.synchronize(); print(f"build {time.time()-t0:.1f}s weights {ranks[0].weights.nbytes/1e9:.2f} GB", flush=True)
slots = [admit(ranks, i, [1, 2, 3], max_ctx=ctx + 200) for i in range(maxb)]
ranks[0].slots.pos[:] = ctx  # pretend ctx tokens of (zero) KV are resident
ex = ranks[0].executor
wbytes = ranks[0].weights.nbytes - geom.vocab * geom.hidden * 2  # embedding rows are gathered, not streamed
for B in batches:
    bk = ex.bucket(B)
    runner.set_rows(bk, slots[:B])
    runner.step(bk, 1)
    runner.capture(bk)
    runner.step(bk, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record(); runner.step(bk, n); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    kv = B * (ctx + 20) * geom.kv_bytes_per_token
    print(f"B={B:4d} bucket={bk} step {ms:.3f} ms  kernels/step {runner.kernels_per_step(bk)}  "
          f"weights+kv {(wbytes+kv)/1e9:.2f} GB -> {(wbytes+kv)/ms/1e6:.0f} GB/s", flush=True)
    ranks[0].slots.pos[:] = ctx
