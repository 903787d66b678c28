"""Dev probe for ncu: one projection GEMM launch per family (QKV, O, gate/up, down) of a TP1
Qwen2.5-7B rank at batch B (default 64), as the decode step issues them (tps_linear with the
step's split-K choice), after warm-up launches on other layers.

ncu --set full -k regex:gemm_swapab -s <warm launches> -c 4 python tools/ncu_gemm_traffic.py [B]
then: python tools/ncu_gemm_traffic.py --summarise <csv> [B]  -> profiles/r2/ncu_traffic.json
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

WARM = 8  # launches before the captured four (ncu -s)
FAMS = ("w_qkv", "w_o", "w_gu", "w_d")


def launch(B):
    import torch
    from paper_2605_23945_b200 import _native as nat
    from paper_2605_23945_b200.models import geometry
    from paper_2605_23945_b200.profiler import loopback_rank
    geom = geometry("qwen2.5-7b")
    r, _ = loopback_rank(geom, 1, B, B, 1024, B * 18)
    ex = r.executor
    xs = {"w_qkv": ex.xn, "w_o": ex.attn, "w_gu": ex.xn, "w_d": ex.act}
    lib = nat.lib()
    st = torch.cuda.current_stream().cuda_stream

    def one(layer, fam):
        w = ex.w[(layer, fam)]
        n, k = w.shape
        x = xs[fam]
        s = lib.tps_linear_splits(n, k, B)
        nat.check(lib.tps_linear(w.data_ptr(), n, k, k, x.data_ptr(), B, x.shape[0], x.shape[1], ex.ws.data_ptr(), s, st))
        return n, k, s
    for i in range(WARM):
        one(2 + i // 4, FAMS[i % 4])
    torch.cuda.synchronize()
    meta = {}
    for fam in FAMS:
        meta[fam] = one(1, fam)
    torch.cuda.synchronize()
    print(json.dumps(meta))


def summarise(path, B):
    from tools.ncu_summary import load
    per, names = load(path)
    ids = sorted(i for i in per if names[i].startswith("tps::gemm") or "gemm_swapab" in names[i])[:4]
    H, F, qkv = 3584, 18944, 4608
    shapes = {"w_qkv": (qkv, H), "w_o": (H, H), "w_gu": (2 * F, H), "w_d": (H, F)}
    out, tot_d, tot_a = {}, 0.0, 0.0
    for fam, i in zip(FAMS, ids):
        n, k = shapes[fam]
        alg = n * k * 2 + B * k * 2 + B * n * 4
        d = per[i].get("dram__bytes_read.sum", 0.0) + per[i].get("dram__bytes_write.sum", 0.0)
        out[fam] = {"dram_bytes": d, "algorithmic_bytes": alg, "ratio": d / alg,
                    "time_us": per[i].get("gpu__time_duration.sum", 0.0) / 1e3}
        tot_d += d
        tot_a += alg
    rec = {"gemm_swapab_kernel": {
        "per_family_B%d" % B: out, "dram_bytes_per_launch": tot_d / len(out),
        "algorithmic_bytes_per_launch": tot_a / len(out),
        "note": (f"ncu --set full dram read+write per launch, mean over one QKV / O / gate-up(+SiLU) / down "
                 f"launch of a Qwen2.5-7B TP1 rank at B={B} (split-K partials included), vs "
                 f"{tot_a / len(out):.0f} algorithmic bytes per launch; profiles/r2/ncu_traffic.json")}}
    os.makedirs("profiles/r2", exist_ok=True)
    with open("profiles/r2/ncu_traffic.json", "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--summarise"]:
        summarise(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 64)
    else:
        launch(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
