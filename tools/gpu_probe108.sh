for i in 1 2 3; do TPS_ATTN_CLUSTER_EARLY=1 timeout 900 python -m pytest tests/test_gpu_decode.py -q 2>&1 | tail -2; done
for e in 0 1; do TPS_ATTN_CLUSTER_EARLY=$e timeout 600 python tools/solo_step.py qwen2.5-7b 8 1,2,8 2048 2>&1 | grep -v watchdog; done
