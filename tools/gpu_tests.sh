timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "silu_cluster" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for v in 0 1; do TPS_SILU_CLUSTER=$v timeout 600 python tools/solo_step.py qwen2.5-7b 4,8 1,8,16,64 2048 2>&1 | grep -v watchdog; done
