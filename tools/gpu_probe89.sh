timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "qkv_rope_in_kernel" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
for c in 8 16; do TPS_QKV_CLUSTER=$c timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,16,64 2048 2>&1 | grep -v watchdog; done
TPS_QKV_CLUSTER=0 timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,16,64 2048 2>&1 | grep -v watchdog
