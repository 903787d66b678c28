"""Dev probe: paged attention time vs split count and kernel (graph-captured, KV > L2)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
nat.init_device(0)
lib = nat.lib()
L, nkv, nq, D = 28, 4, 28, 128
cases = ((64, 2048), (64, 512), (32, 4096), (16, 4096), (4, 8192), (1, 8192), (1, 2048), (128, 1024), (256, 1024))
if len(sys.argv) > 1:
    cases = [a for a in sys.argv[1:]]
for case in cases:
    ragged = isinstance(case, str) and case.endswith("r")
    B, ctx = (tuple(int(v) for v in case.rstrip("r").split("x")) if isinstance(case, str) else case)
    pages = (ctx + 63) // 64
    num_pages = B * pages
    Lr = max(2, min(L, int(4e9 // (num_pages * nkv * 64 * D * 4))))
    kv = torch.randn(Lr, 2, num_pages, nkv, 64, D, device="cuda").bfloat16()
    pt = torch.arange(num_pages, dtype=torch.int32, device="cuda").view(B, pages)
    rs = torch.arange(B, dtype=torch.int32, device="cuda")
    pos = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
    if ragged:  # contexts uniform in [1, ctx] (seeded), one row at the maximum
        g = torch.Generator().manual_seed(0)
        pos = torch.randint(0, ctx, (B,), generator=g, dtype=torch.int32)
        pos[0] = ctx - 1
        pos = pos.cuda()
    q = torch.randn(B, nq, D, device="cuda").bfloat16()
    out = torch.empty(B, nq, D, device="cuda", dtype=torch.bfloat16)
    ctr = torch.zeros(B * nkv, dtype=torch.int32, device="cuda")
    ws = max(lib.tps_attn_workspace(B, nq, D, 0), B * nq * 128 * D)
    pm = torch.empty(ws // D, device="cuda"); pl = torch.empty_like(pm)
    po = torch.empty(ws, device="cuda")
    default = lib.tps_attn_splits(B, nkv, pages)
    torch.cuda.synchronize()  # inputs are built on the default stream; the probe launches on side streams
    res = []
    import os
    nss = [int(v) for v in os.environ.get("SWEEP_NS", "0,1,2,3,4,6,8,12,16,24,32").split(",")]
    for tma in (0,):
        for ns in sorted(set(nss) | {default}):
            if ns > pages:
                continue
            st = torch.cuda.Stream()
            def run(l):
                nat.check(lib.tps_paged_attention(q.data_ptr(), kv[l, 0].data_ptr(), kv[l, 1].data_ptr(), rs.data_ptr(),
                                                  pos.data_ptr(), None, pt.data_ptr(), pages, B, nq, nkv, D, ns,
                                                  pm.data_ptr(), pl.data_ptr(), po.data_ptr(), ctr.data_ptr(),
                                                  out.data_ptr(), None, 0, 0, None, None, None, st.cuda_stream))
            with torch.cuda.stream(st):
                for l in range(Lr): run(l)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for l in range(Lr): run(l)
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): g.replay()
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * Lr)
            byt = int((pos.long() + 1).sum()) * nkv * D * 2 * 2
            res.append((us, tma, ns))
            print(f"B={B} ctx={ctx}{'r' if ragged else ''} nsplit={ns}{'*' if ns == default else ''}: {us:.1f} us/layer, "
                  f"{byt/us/1e3:.0f} GB/s", flush=True)
    best = min(res)
    print(f"BEST B={B} ctx={ctx}{'r' if ragged else ''}: nsplit={best[2]} {best[0]:.1f} us (default {default})", flush=True)
    del kv
