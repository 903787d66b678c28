mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_step -c 1 -s 1 -o gpurun_out/persist_tp8b1_v3 python tools/persist_once.py qwen2.5-7b 8 1 2048 2 > gpurun_out/ncu1.log 2>&1
tail -2 gpurun_out/ncu1.log
