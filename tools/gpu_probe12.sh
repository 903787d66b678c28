NCU=/usr/local/cuda/bin/ncu
K='regex:^(gemm|paged|add_norm|qkv|reduce|argmax|embed|epoch|silu|attn)'
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --launch-skip 286 --launch-count 286 --csv --log-file gpurun_out/solo_tp8_b1.csv timeout 300 python tools/solo_once.py qwen2.5-7b 8 1 2048 2 > gpurun_out/solo_once.log 2>&1
python tools/ncu_summary.py gpurun_out/solo_tp8_b1.csv
python - <<'PY'
import sys; sys.path.insert(0, "tools")
from ncu_summary import load
per, names = load("gpurun_out/solo_tp8_b1.csv")
ids = sorted(per)[:12]
for i in ids:
    print(names[i], round(per[i]["gpu__time_duration.sum"]/1e3, 2), "us", round((per[i].get("dram__bytes_read.sum",0)+per[i].get("dram__bytes_write.sum",0))/1e6, 2), "MB")
PY
