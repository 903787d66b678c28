timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "argmax_epilogue" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_coordinator.py -x -q 2>&1 | tail -2
for v in 0 1; do TPS_LM_ARGMAX=$v timeout 600 python tools/solo_step.py qwen2.5-7b 1 1,16,64 2048 2>&1 | grep -v watchdog; done
