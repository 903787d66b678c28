import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.executor import FUSE_ROWS, FUSE_SOURCES
nat.init_device(0)
lib = nat.lib()
H = 3584
for (K, S, tp) in ((1792, 5, 2), (512, 2, 8), (1792, 5, 1), (1024, 4, 4)):
    ll = torch.zeros((2, FUSE_SOURCES, FUSE_ROWS, H), dtype=torch.int64, device="cuda")
    epoch = torch.ones(1, dtype=torch.int64, device="cuda")
    w = (torch.randn(H, K, device="cuda") * 0.05).bfloat16()
    x = torch.randn(1, K, device="cuda").bfloat16()
    slot = FUSE_ROWS * H * 8
    dsts = [ll.data_ptr() + q * S * slot for q in range(tp)]
    nat.check(lib.tps_linear_push_ll(w.data_ptr(), H, K, K, x.data_ptr(), 1, 1, K, nat.ptr_array(dsts), len(dsts),
                                     FUSE_ROWS * H, S, epoch.data_ptr(), 57, 0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    tags = (ll[0, :, 0] >> 32)
    print(K, S, tp, "slots with tag 57 per source:", [(int((tags[i] == 57).sum())) for i in range(FUSE_SOURCES)])
