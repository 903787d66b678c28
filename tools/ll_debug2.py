import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank
from paper_2605_23945_b200.executor import FUSE_ROWS, FUSE_SOURCES
lib = nat.lib()
geom = geometry("qwen2.5-7b")
r, runner = loopback_rank(geom, 2, 1, 1, 2304, 40)
ex = r.executor; cm = ex.comm
w = ex.w[(0, "w_o")]; x = ex.attn
n, k = w.shape
S = ex.fused_splits("w_o", 1)
H = geom.hidden
dsts = [cm.ll_slot(base, 0, q, S) for q, base in enumerate(cm.peer_ll)]
print("w", w.shape, w.stride(), "x", x.shape, x.stride(), "S", S, "dsts", [hex(d - cm.ll.data_ptr()) for d in dsts])
nat.check(lib.tps_linear_push_ll(w.data_ptr(), n, k, k, x.data_ptr(), 1, x.shape[0], x.shape[1], nat.ptr_array(dsts),
                                 len(dsts), FUSE_ROWS * H, S, cm.epoch.data_ptr(), cm.n_phases, 0,
                                 torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
tags = cm.ll[0, :, 0] >> 32
print("tags==57 per slot:", [int((tags[i] == 57).sum()) for i in range(FUSE_SOURCES)])
# full eager step with the consumers skipped: inspect what the step leaves in the LL slots
from paper_2605_23945_b200.group import admit
r2, runner2 = loopback_rank(geom, 2, 1, 1, 2304, 40)
ex2 = r2.executor; cm2 = ex2.comm
slots = [admit([r2], 0, [1, 2, 3], max_ctx=2200)]
r2.slots.pos[:] = 2048
runner2.set_rows(1, slots)
ex2.skip = frozenset({"add_norm"})
runner2.step(1, 1)
torch.cuda.synchronize()
for par in (0, 1):
    tags = cm2.ll[par, :, 0] >> 32
    print("par", par, "distinct tags per slot:", [sorted(set(tags[i].tolist()))[:4] for i in range(10)])
