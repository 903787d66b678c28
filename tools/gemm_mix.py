"""Dev probe: per-layer time of the 4 projections chained in step order (graph), with/without the fused push."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
tps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 8]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
geom = geometry(name)
lib = nat.lib()


def run(issue, label, L):
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g.capture_begin()
        issue(st.cuda_stream)
        g.capture_end()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) * 1e3 / (5 * L):7.2f} us/layer", flush=True)


for tp in tps:
    r, runner = loopback_rank(geom, tp, max(B, 16), max(B, 16), 4096, 64)
    ex = r.executor
    cm = ex.comm
    xs = {"w_qkv": ex.xn, "w_o": ex.attn, "w_gu": ex.xn, "w_d": ex.act}
    L = geom.num_layers

    def lin(st, fam, l, push):
        w = ex.w[(l, fam)]
        n, k = w.shape
        x = xs[fam]
        if push and cm is not None:
            S = ex.fused_splits(fam, B)
            dsts = [cm.frecv_slot(b, 0, 0, S) for b in cm.peer_frecv]
            sigs = [p for p in cm.peer_ctr]
            nat.check(lib.tps_linear_push(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                          nat.ptr_array(dsts), len(dsts), 64 * geom.hidden, S,
                                          nat.ptr_array(sigs), len(sigs), cm.done.data_ptr(), st))
        else:
            s = lib.tps_linear_splits(n, k, B)
            nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1],
                                     ex.ws.data_ptr(), s, st))

    for push in (False, True):
        def issue(st, push=push):
            for l in range(L):
                for fam in ("w_qkv", "w_o", "w_gu", "w_d"):
                    lin(st, fam, l, push and fam in ("w_o", "w_d"))
        run(issue, f"tp={tp} B={B} 4-GEMM layer chain push={push}", L)
    for fam in ("w_qkv", "w_o", "w_gu", "w_d"):
        def issue(st, fam=fam):
            for l in range(L):
                lin(st, fam, l, False)
        run(issue, f"tp={tp} B={B} {fam} only", L)
    del r, runner
    torch.cuda.empty_cache()
