mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tp8_b1.csv python tools/solo_once.py qwen2.5-7b 8 1 2048 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tp1_b64.csv python tools/solo_once.py qwen2.5-7b 1 64 2048 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_swapab --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_full_cluster_ll_tp8 python tools/solo_once.py qwen2.5-7b 8 1 2048 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_prefill --launch-count 1 -o gpurun_out/ncu_full_prefill_attn python tools/trace_prefill.py qwen2.5-7b 256 > /dev/null 2>&1
ls -la gpurun_out/ | grep ncu
