"""Dev probe: in-chain timeline of one chunked-prefill step (512 rows) on one rank.

python tools/trace_prefill.py <model> <ctx> [tp]  (tp > 1: loopback rank, tools/solo_step.py)"""
import collections, sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

KIND = {1: "embed", 2: "add_norm", 3: "reduce_push", 4: "qkv_rope", 5: "silu_mul", 6: "argmax1", 7: "argmax2",
        8: "epoch", 9: "gemm", 10: "gemm_silu", 11: "attn_split", 12: "attn_combine", 13: "attn_bal", 14: "attn_prefill", 15: "gemm_push", 16: "gemv"}
name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 256
tp = int(sys.argv[3]) if len(sys.argv) > 3 else 1
R = 512
geom = geometry(name)
nb = 64
r, runner = loopback_rank(geom, tp, nb, nb, ctx + 256, nb * ((ctx + 256) // 64 + 2), prefill_rows=R)
ex = r.executor
ppl = (ctx + 64) // 64 + 1
r.slots.page_table[:nb, :ppl].copy_(torch.arange(nb * ppl, dtype=torch.int32).view(nb, ppl))
rs = torch.tensor([i % nb for i in range(R)], dtype=torch.int32)
rp = torch.tensor([ctx - R // nb + i // nb for i in range(R)], dtype=torch.int32)
ex.set_prefill_rows(rs, rp)
key = ("prefill", R)
runner._capture_key(key, lambda s_: runner._issue_prefill(R, s_))
g = runner.graphs[key]
g.replay(); g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"prefill step R={R} ctx~{ctx}: {e0.elapsed_time(e1):.3f} ms")
cap = 2048
rec = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
nat.check(nat.lib().tps_trace_enable(rec.data_ptr(), ctr.data_ptr(), cap))
g.replay(); torch.cuda.synchronize()
nat.check(nat.lib().tps_trace_enable(None, None, 0))
n = int(ctr.item())
R_ = rec[:4 * n].view(n, 4).cpu().tolist()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
prev = None
for kind, te, tw, tx in R_:
    a = agg[KIND.get(kind, str(kind))]
    a[0] += 1; a[1] += (tx - tw) / 1e3
    if prev is not None: a[2] += (tw - prev) / 1e3
    prev = tx
for k, (c, w, gg) in sorted(agg.items(), key=lambda x: -(x[1][1] + x[1][2])):
    print(f"{k:12s} {c:4d} work {w / c:8.2f} us  wait {gg / c:6.2f} us  total {w + gg:8.1f} us")
names = []
for kind, te, tw, tx in R_[:10]:
    print(f"  {KIND.get(kind, kind):12s} work {(tx - tw) / 1e3:8.2f} us")
