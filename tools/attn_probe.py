"""Dev probe: paged attention bandwidth alone (layers cycled, KV > L2)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
nat.init_device(0)
lib = nat.lib()
L, nkv, nq, D = 28, 4, 28, 128
for B, ctx in ((64, 2048), (64, 512), (16, 4096), (1, 8192), (1, 2048)):
    pages = (ctx + 63) // 64
    num_pages = B * pages
    kv = torch.randn(L, 2, num_pages, nkv, 64, D, device="cuda").bfloat16()
    pt = torch.arange(num_pages, dtype=torch.int32, device="cuda").view(B, pages)
    rs = torch.arange(B, dtype=torch.int32, device="cuda")
    pos = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(B, nq, D, device="cuda").bfloat16()
    ns = 0  # page-balanced schedule
    ws = lib.tps_attn_workspace(B, nq, D, ns)
    pm = torch.empty(ws // D, device="cuda"); pl = torch.empty_like(pm)
    po = torch.empty(ws, device="cuda"); ctr = torch.zeros(B * nkv, dtype=torch.int32, device="cuda")
    out = torch.empty(B, nq, D, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    def run(l):
        lib.tps_paged_attention(q.data_ptr(), kv[l, 0].data_ptr(), kv[l, 1].data_ptr(), rs.data_ptr(), pos.data_ptr(),
                                None, pt.data_ptr(), pages, B, nq, nkv, D, ns, pm.data_ptr(), pl.data_ptr(),
                                po.data_ptr(), ctr.data_ptr(), out.data_ptr(), None, 0, 0, None, None, None, st)
    for tma in (0,):
        for l in range(L): run(l)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for rep in range(3):
            for l in range(L): run(l)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (3 * L)
        byt = B * ctx * nkv * D * 2 * 2
        print(f"tma={tma} B={B} ctx={ctx} nsplit={ns}: {us:.1f} us/layer, {byt/us/1e3:.0f} GB/s", flush=True)
    del kv
