timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention 2>&1 | tail -2
timeout 900 python tools/solo_step.py qwen2.5-7b 1,4,8 1,2 2048 "" 2>&1 | grep -v watchdog
timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048 2>&1 | sed -n 1,10p
