"""tps_kv_move_items on a B200 vs its CPU restatement (oracle/reshard_ref.expand_kv_moves).

The Switch Executor describes KV migration as one move per (sample, kv-head run) and the
device expands the moves into copy items from the page tables; the item table must equal the
oracle's expansion of the same descriptors item for item, out-of-range pages must yield empty
items and be counted, and executing the items must move the pages bit-exactly.
"""

import numpy as np
import pytest
import torch

from oracle.reshard_ref import ByteMemory, expand_kv_moves
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.models import geometry, rank_shard
from paper_2605_23945_b200.switch_executor import Layout, pack_kv_moves, plan_kv_moves

pytestmark = pytest.mark.gpu


class _DevMem(ByteMemory):
    """ByteMemory view of device page tables (copied to the host once) for the oracle."""

    def __init__(self, tables: dict[int, np.ndarray]):
        super().__init__()
        self.bufs = [(ptr, arr.view(np.uint8).ravel()) for ptr, arr in tables.items()]


@pytest.mark.parametrize("t0,t1", [(1, 2), (2, 8), (8, 2), (1, 8)])
def test_kv_move_items_match_oracle_and_copy_bit_exact(t0, t1):
    geom = geometry("qwen2.5-7b")
    world, L, D = 8, 3, geom.head_dim  # 3 layers of the real per-layer KV shape
    chunk = 64 * D * 2
    nat.init_device(0)
    old, new = Layout(t0, world), Layout(t1, world)
    rng = np.random.default_rng(t0 * 10 + t1)
    dev = torch.device("cuda:0")
    P, npg_old, npg_new, slots = 40, 256, 300, 8
    n_samples = 6
    ctx = rng.integers(1, P * 64, n_samples)
    og = rng.integers(0, old.dp, n_samples)
    oslot = np.arange(n_samples) + 1
    src, keep = {}, []
    tables = {}
    perm = rng.permutation(npg_old).astype(np.int32)
    for r in range(world):
        sh = rank_shard(geom, t0, r % t0)
        kv = torch.randint(-30000, 30000, (L, 2, npg_old, sh.n_kv, 64, D), dtype=torch.int16, device=dev)
        pt = torch.zeros((slots, P), dtype=torch.int32)
        for i in range(n_samples):
            pt[oslot[i]] = torch.from_numpy(perm[i * P:(i + 1) * P])
        ptd = pt.to(dev)
        keep += [kv, ptd]
        tables[ptd.data_ptr()] = pt.numpy()
        src[r] = {"kv": kv.data_ptr(), "pt": ptd.data_ptr(), "np": npg_old, "nkv": sh.n_kv, "t": kv}
    for dst in (0, world - 1):
        sh = rank_shard(geom, t1, dst % t1)
        mine = [i for i in range(n_samples) if i % new.dp == new.group_of(dst)]
        nslot = np.arange(len(mine)) + 2
        pt = torch.zeros((slots, P), dtype=torch.int32)
        dperm = rng.permutation(npg_new).astype(np.int32)
        for j in range(len(mine)):
            pt[nslot[j]] = torch.from_numpy(dperm[j * P:(j + 1) * P])
        ptd = pt.to(dev)
        tables[ptd.data_ptr()] = pt.numpy()
        pool = torch.zeros((L, 2, npg_new, sh.n_kv, 64, D), dtype=torch.int16, device=dev)
        moves = plan_kv_moves(geom, old, new, dst, og[mine], oslot[mine], nslot, ctx[mine])
        packed, n_items = pack_kv_moves(geom, moves, src, ptd.data_ptr(), 4 * P)
        # the geometry's layer count is 28; the pools here hold 3 layers
        per = 2 * L * packed["n_pages"].astype(np.int64)
        packed["first_item"] = np.cumsum(per) - per
        n_items = int(per.sum())
        ref = expand_kv_moves(_DevMem(tables), packed, pool.data_ptr(), npg_new, sh.n_kv, L, chunk)
        dmov = torch.from_numpy(packed.view(np.uint8).copy()).to(dev)
        items = torch.zeros((n_items, 4), dtype=torch.int64, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        nat.check(nat.lib().tps_kv_move_items(dmov.data_ptr(), len(packed), n_items, pool.data_ptr(), npg_new,
                                              sh.n_kv, chunk, items.data_ptr(), bad.data_ptr(), 0), "kv_move_items")
        torch.cuda.synchronize()
        assert int(bad.item()) == 0
        assert np.array_equal(items.cpu().numpy(), ref)
        nat.check(nat.lib().tps_copy_items(items.data_ptr(), n_items, 1, 0, 0), "copy_items")
        torch.cuda.synchronize()
        for m in moves:
            s_rank, s_slot, s_head, d_slot, d_head, nh, npg = (int(x) for x in m)
            spages = torch.from_numpy(tables[src[s_rank]["pt"]][s_slot][:npg]).long().to(dev)
            dpages = pt[d_slot][:npg].long().to(dev)
            a = src[s_rank]["t"][:, :, spages, s_head:s_head + nh]
            b = pool[:, :, dpages, d_head:d_head + nh]
            assert torch.equal(a, b), (t0, t1, dst, m)


def test_kv_move_items_flags_out_of_range_pages():
    dev = torch.device("cuda:0")
    nat.init_device(0)
    from paper_2605_23945_b200.switch_executor import KV_MOVE_DTYPE
    kv = torch.zeros(2 * 2 * 4 * 64 * 64, dtype=torch.int16, device=dev)
    pt = torch.tensor([0, 7, 1], dtype=torch.int32, device=dev)  # page 7 is outside a 4-page pool
    mv = np.zeros(1, dtype=KV_MOVE_DTYPE)
    mv["src_kv"], mv["src_pages"], mv["dst_pages"] = kv.data_ptr(), pt.data_ptr(), pt.data_ptr()
    mv["src_num_pages"], mv["src_nkv"], mv["n_heads"], mv["n_pages"] = 4, 1, 1, 3
    dmov = torch.from_numpy(mv.view(np.uint8).copy()).to(dev)
    n = 2 * 1 * 3
    items = torch.full((n, 4), -1, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    nat.check(nat.lib().tps_kv_move_items(dmov.data_ptr(), 1, n, kv.data_ptr(), 4, 1, 64 * 64 * 2, items.data_ptr(),
                                          bad.data_ptr(), 0), "kv_move_items")
    torch.cuda.synchronize()
    got = items.cpu()
    assert int(bad.item()) == 2  # page 7 in K and in V of the one layer
    assert int((got[:, 2] == 0).sum()) == 2
