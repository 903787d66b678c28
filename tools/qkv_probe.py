"""Dev probe: QKV projection finished in-kernel (tps_linear_qkv_rope) vs tps_linear +
tps_qkv_rope_append, timed as 50-launch CUDA graphs (PDL chain) at decode shapes."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat

nat.init_device(0)
lib = nat.lib()
st = torch.cuda.Stream()
for (nq, nkv, k, b) in [(28, 4, 3584, 64), (28, 4, 3584, 16), (28, 4, 3584, 1), (4, 1, 3584, 1), (4, 1, 3584, 16)]:
    D, P, max_pages = 128, 64, 40
    n = (nq + 2 * nkv) * D
    S = lib.tps_qkv_fused_splits(n, k, b)
    S0 = lib.tps_linear_splits(n, k, b)
    ws_ = [(torch.randn(n, k, device="cuda") * 0.05).bfloat16() for _ in range(8)]  # > L2 cycling
    x = torch.randn(b, k, device="cuda").bfloat16()
    bvec = torch.zeros(n, device="cuda").bfloat16()
    slots = b
    pos = torch.full((slots,), 1000, dtype=torch.int32, device="cuda")
    rs = torch.arange(b, dtype=torch.int32, device="cuda")
    pt = torch.arange(slots * max_pages, dtype=torch.int32, device="cuda").view(slots, max_pages)
    cos = torch.ones(P * max_pages, D // 2, device="cuda")
    sin = torch.zeros_like(cos)
    q = torch.zeros(b, nq, D, device="cuda").bfloat16()
    kc = torch.zeros(slots * max_pages, nkv, P, D, device="cuda").bfloat16()
    vc = torch.zeros_like(kc)
    wsp = torch.zeros(max(S, S0), b, n, device="cuda")

    def fused(w):
        nat.check(lib.tps_linear_qkv_rope(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k, bvec.data_ptr(), rs.data_ptr(),
                                          pos.data_ptr(), None, pt.data_ptr(), max_pages, cos.data_ptr(),
                                          sin.data_ptr(), nq, nkv, D, P, q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                                          st.cuda_stream))

    def split(w, s):
        nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k, wsp.data_ptr(), s, st.cuda_stream))
        nat.check(lib.tps_qkv_rope_append(wsp.data_ptr(), s, b * n, bvec.data_ptr(), rs.data_ptr(), pos.data_ptr(),
                                          None, pt.data_ptr(), max_pages, cos.data_ptr(), sin.data_ptr(), b, nq, nkv,
                                          D, P, q.data_ptr(), kc.data_ptr(), vc.data_ptr(), st.cuda_stream))

    def gemm_only(w, s):
        nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), b, b, k, wsp.data_ptr(), s, st.cuda_stream))

    res = {}
    for name, fn in [("fused", lambda w: fused(w)), (f"linear(S={S0})+rope", lambda w: split(w, S0)),
                     (f"linear(S={S})+rope", lambda w: split(w, S)), (f"linear(S={S0})", lambda w: gemm_only(w, S0))]:
        with torch.cuda.stream(st):
            for i in range(3):
                fn(ws_[i % 8])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(48):
                    fn(ws_[i % 8])
            g.replay(); g.replay()
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); g.replay(); e1.record(st); st.synchronize()
            res[name] = e0.elapsed_time(e1) * 1e3 / 48
    print(f"nq={nq} nkv={nkv} n={n} k={k} b={b} S_fused={S}: " +
          "  ".join(f"{k_}: {v:.2f} us" for k_, v in res.items()), flush=True)
