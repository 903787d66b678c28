timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_coordinator.py -x -q 2>&1 | tail -2
for t in 0 1; do TPS_ATTN_TMA_BAL=$t timeout 600 python tools/solo_step.py qwen2.5-7b 4,8 12,16,32,64 2048 2>&1 | grep -v watchdog | sed "s/^/bal_tma=$t /"; done
