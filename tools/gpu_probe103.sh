timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "push_ll_cluster" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_coordinator.py -x -q 2>&1 | tail -3
for r in 0 16 64; do echo "== LL cluster rows $r"; TPS_LL_CLUSTER_ROWS=$r timeout 600 python tools/solo_step.py qwen2.5-7b 2,4,8 1,8,16,32,64 2048 2>&1 | grep -v watchdog; done
