for v in 0 1; do echo "== cluster linear $v"; TPS_CLUSTER_LINEAR=$v timeout 600 python tools/solo_step.py qwen2.5-7b 1,2,8 1,16,64 2048 2>&1 | grep -v watchdog; done
TPS_CLUSTER_LINEAR=1 timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
