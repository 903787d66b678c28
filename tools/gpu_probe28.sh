CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/solo_step.py qwen2.5-7b 2 1 2048 "" > gpurun_out/tp2dbg.log 2>&1
grep "tps watchdog" gpurun_out/tp2dbg.log | awk '{print $5, $6, $7, $8, $10}' | sort | uniq -c | head; grep "tps watchdog" gpurun_out/tp2dbg.log | head -3
