for cs in 16 8 4; do for c in 512 2048 8192; do echo "== cluster $cs ctx $c"; TPS_ATTN_CLUSTER_SIZE=$cs timeout 600 python tools/solo_step.py qwen2.5-7b 8 1,2,8 $c 2>&1 | grep -v watchdog; done; done
