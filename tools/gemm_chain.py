"""Dev probe: per-launch time of each projection family in a graph of 28 (distinct-weight) launches."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
tps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 8]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
forced = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else []
geom = geometry(name)
lib = nat.lib()
for tp in tps:
    r, runner = loopback_rank(geom, tp, max(B, 16), max(B, 16), 4096, 64)
    ex = r.executor
    xs = {"w_qkv": ex.xn, "w_o": ex.attn, "w_gu": ex.xn, "w_d": ex.act}
    for fam in ("w_qkv", "w_o", "w_gu", "w_d"):
        w0 = ex.w[(0, fam)]
        n, k = w0.shape
        x = xs[fam]
        for s in ([lib.tps_linear_splits(n, k, B)] + forced):
            if s > (k + 63) // 64:
                continue
            ws = torch.zeros(s * B * n, device="cuda")
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                g.capture_begin()
                for l in range(geom.num_layers):
                    w = ex.w[(l, fam)]
                    lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1], ws.data_ptr(), s,
                                   st.cuda_stream)
                g.capture_end()
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * geom.num_layers)
            print(f"tp={tp} B={B} {fam:6s} n={n:6d} k={k:6d} splits={s:2d}: {us:6.2f} us/launch "
                  f"{n * k * 2 / us / 1e3:7.0f} GB/s", flush=True)
    del r, runner
    torch.cuda.empty_cache()
