for mb in 0 40 80; do echo "== L2 prefetch ${mb} MB"; TPS_L2_PREFETCH_MB=$mb timeout 600 python tools/solo_step.py qwen2.5-7b 2,4,8 1,16,64 2048 2>&1 | grep -v watchdog; done
