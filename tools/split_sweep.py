"""Dev probe: projection GEMM time vs split-K count (weights cycled over layers, > L2)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
nat.init_device(0)
lib = nat.lib()
L = 28
shapes = {"qkv": (4608, 3584), "o": (3584, 3584), "gu": (37888, 3584), "down": (3584, 18944), "lm": (152064, 3584)}
st = torch.cuda.current_stream()
for name, (n, k) in shapes.items():
    nl = L if name != "lm" else 4
    ws = [torch.randn(n, k, device="cuda").bfloat16() for _ in range(nl)]
    x = torch.randn(256, k, device="cuda").bfloat16()
    out = torch.empty(32 * 256 * n if n < 40000 else 4 * 256 * n, device="cuda")
    for B in (1, 16, 64):
        res = []
        smax = min(32, (k + 63) // 64) if n < 40000 else 4
        for s in sorted({1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32} & set(range(1, smax + 1))):
            for w in ws[:2]:
                lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, 256, k, out.data_ptr(), s, st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for w in ws:
                lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, 256, k, out.data_ptr(), s, st.cuda_stream)
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / nl
            res.append((us, s))
        best = min(res)
        print(f"{name} B={B} heuristic={lib.tps_linear_splits(n,k,B)} best s={best[1]} {best[0]:.2f}us "
              f"({n*k*2/best[0]/1e3:.0f} GB/s) | " + " ".join(f"{s}:{us:.1f}" for us, s in res), flush=True)
    del ws
