"""Dev probe: per-launch latency of single kernels replayed in a CUDA graph (PDL on/off)."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat

nat.init_device(0)
lib = nat.lib()
H = 3584
resid = torch.zeros(64, H, device="cuda")
xn = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
wn = torch.ones(H, dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(40 * 64 * H, device="cuda")
epoch = torch.ones(1, dtype=torch.int64, device="cuda")
N = 200


def timed(issue, label):
    for pdl in (1, 0):
        lib.tps_set_pdl(pdl)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(N):
                issue(s.cuda_stream)
            g.capture_end()
        g.replay(); g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
        print(f"{label:40s} pdl={pdl}: {e0.elapsed_time(e1) * 1e3 / (2 * N):6.2f} us/launch", flush=True)
    lib.tps_set_pdl(1)


timed(lambda st: lib.tps_epoch_advance(epoch.data_ptr(), st), "epoch_advance (1 thread)")
for B in (1, 64):
    for nsrc in (0, 4, 40):
        timed(lambda st: lib.tps_add_norm(resid.data_ptr(), ws.data_ptr() if nsrc else None, nsrc, 64 * H if nsrc else 0,
                                          None, wn.data_ptr(), ctypes.c_float(1e-6), H, B, xn.data_ptr(), H, st),
              f"add_norm B={B} nsrc={nsrc}")
# alternating epoch_advance and add_norm
def alt(st):
    lib.tps_add_norm(resid.data_ptr(), ws.data_ptr(), 4, 64 * H, None, wn.data_ptr(), ctypes.c_float(1e-6), H, 1,
                     xn.data_ptr(), H, st)
    lib.tps_epoch_advance(epoch.data_ptr(), st)
timed(alt, "add_norm(B=1,4 src) + epoch_advance pair")
# small GEMMs back to back (TP8 shapes) and a big one
for (n, k, B) in ((768, 3584, 1), (3584, 512, 1), (4736, 3584, 1), (3584, 2368, 1), (37888, 3584, 1)):
    w = torch.zeros(n, k, dtype=torch.bfloat16, device="cuda")
    x = torch.zeros(64, k, dtype=torch.bfloat16, device="cuda")
    s_ = lib.tps_linear_splits(n, k, B)
    out = torch.zeros(s_ * 64 * n, device="cuda")
    timed(lambda st: lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, 64, k, out.data_ptr(), s_, st),
          f"linear n={n} k={k} B={B} splits={s_} ({n*k*2/1e6:.1f} MB)")
    del w
