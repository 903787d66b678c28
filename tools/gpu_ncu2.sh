NCU=/usr/local/cuda/bin/ncu
K='regex:^(gemm|paged|add_norm|qkv|reduce|argmax|embed|epoch|silu|attn)'
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --launch-skip 258 --launch-count 258 --csv --log-file gpurun_out/ncu_solo_tp8_b1.csv timeout 300 python tools/solo_once.py qwen2.5-7b 8 1 2048 2 > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --launch-skip 229 --launch-count 229 --csv --log-file gpurun_out/ncu_tp1_b64.csv timeout 300 python tools/solo_once.py qwen2.5-7b 1 64 2048 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_solo_tp8_b1.csv > gpurun_out/ncu_solo_tp8_b1_summary.txt
python tools/ncu_summary.py gpurun_out/ncu_tp1_b64.csv > gpurun_out/ncu_tp1_b64_summary.txt
cat gpurun_out/ncu_solo_tp8_b1_summary.txt gpurun_out/ncu_tp1_b64_summary.txt
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_attn_cluster --launch-skip 60 -c 1 -o gpurun_out/ncu_attn_cluster -f python tools/solo_once.py qwen2.5-7b 8 1 4096 2 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:add_norm_cluster --launch-skip 120 -c 1 -o gpurun_out/ncu_addnorm_ll -f python tools/solo_once.py qwen2.5-7b 8 1 2048 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
