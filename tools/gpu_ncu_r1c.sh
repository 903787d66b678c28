mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tp8_b1.csv python tools/solo_once.py qwen2.5-7b 8 1 2048 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tp1_b64.csv python tools/solo_once.py qwen2.5-7b 1 64 2048 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_kernel --launch-skip 30 --launch-count 1 -o gpurun_out/ncu_full_attn_tma_b64 python tools/solo_once.py qwen2.5-7b 1 64 512 2 > /dev/null 2>&1
TPS_ATTN_TMA=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_kernel --launch-skip 30 --launch-count 1 -o gpurun_out/ncu_full_attn_cpasync_b64 python tools/solo_once.py qwen2.5-7b 1 64 512 2 > /dev/null 2>&1
ls gpurun_out | grep ncu
