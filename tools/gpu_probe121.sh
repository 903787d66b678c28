for mb in 0 30 40 150; do echo "== shallow <= $mb MB"; TPS_GEMM_SHALLOW_MB=$mb timeout 600 python tools/solo_step.py qwen2.5-7b 1,2 1,16,64 2048 2>&1 | grep -v watchdog; done
