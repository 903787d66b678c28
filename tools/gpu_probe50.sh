timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 900 python tools/solo_step.py qwen2.5-7b 2,4,8 1,16,48 3072 "" 2>&1 | grep -v watchdog
