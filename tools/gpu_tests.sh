timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kernels.py -x -q -k "argmax or decode or oracle or stochastic or graph" 2>&1 | tail -2
timeout 600 python tools/solo_step.py qwen2.5-7b 1 1,16,64 2048 2>&1 | grep -v watchdog
