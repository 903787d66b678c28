TPS_ATTN_TMA=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -3
TPS_ATTN_TMA=1 timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for t in 0 1; do for c in 512 2048; do TPS_ATTN_TMA=$t timeout 600 python tools/solo_step.py qwen2.5-7b 1 16,64 $c 2>&1 | grep -v watchdog | sed "s/^/tma=$t /"; done; done
