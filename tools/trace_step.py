"""Dev probe: in-chain timeline of one graph-replayed decode step (device step tracer).

python tools/trace_step.py qwen2.5-7b <tp> <B> <ctx>
Per kernel kind: count, mean in-kernel time after its PDL wait (t_exit - t_wait), mean wait
release after the previous kernel's exit (t_wait - prev t_exit), share of the step.
"""
import collections, sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

KIND = {1: "embed", 2: "add_norm", 3: "reduce_push", 4: "qkv_rope", 5: "silu_mul", 6: "argmax1", 7: "argmax2",
        8: "epoch", 9: "gemm", 10: "gemm_silu", 11: "attn_split", 12: "attn_combine", 13: "attn_bal", 14: "attn_prefill", 15: "gemm_push", 16: "gemv"}
name, tp, B, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
geom = geometry(name)
r, runner = loopback_rank(geom, tp, B, B, ctx + 256, B * ((ctx + 256) // 64 + 2))
slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(B)]
r.slots.pos[:] = ctx
bk = r.executor.bucket(B)
runner.set_rows(bk, slots)
runner.step(bk, 1)
runner.capture(bk)
runner.step(bk, 3)
torch.cuda.synchronize()
cap = 4096
rec = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
nat.check(nat.lib().tps_trace_enable(rec.data_ptr(), ctr.data_ptr(), cap))
runner.step(bk, 1)
torch.cuda.synchronize()
nat.check(nat.lib().tps_trace_enable(None, None, 0))
n = int(ctr.item())
R = rec[:4 * n].view(n, 4).cpu().tolist()
t0 = R[0][1]
step = max(x[3] for x in R) - t0
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
prev_exit = None
for kind, te, tw, tx in R:
    a = agg[KIND.get(kind, str(kind))]
    a[0] += 1
    a[1] += (tx - tw) / 1e3
    if prev_exit is not None:
        a[2] += (tw - prev_exit) / 1e3
    prev_exit = tx
print(f"{name} tp={tp} B={B} ctx={ctx}: {n} traced launches, step span {step / 1e3:.1f} us")
print(f"{'kind':14s} {'n':>4s} {'work_us':>9s} {'wait_us':>9s} {'total_us':>9s} {'share':>6s}")
for k, (c, w, g) in sorted(agg.items(), key=lambda x: -(x[1][1] + x[1][2])):
    print(f"{k:14s} {c:4d} {w / c:9.2f} {g / c:9.2f} {w + g:9.1f} {100 * (w + g) * 1e3 / step:5.1f}%")
print("first layer:")
for kind, te, tw, tx in R[:12]:
    print(f"  {KIND.get(kind, kind):12s} entry {(te - t0) / 1e3:8.2f} wait_done {(tw - t0) / 1e3:8.2f} exit {(tx - t0) / 1e3:8.2f}")
