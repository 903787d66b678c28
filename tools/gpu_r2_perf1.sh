mkdir -p gpurun_out
timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,4,8,16 2048 2>&1 | grep -v watchdog | tail -16
TPS_PERSIST=0 timeout 900 python tools/solo_step.py qwen2.5-7b 8 1,16 2048 2>&1 | grep -v watchdog | tail -2
timeout 1800 python -m pytest tests/test_gpu_decode_fullshape.py -q -s 2>&1 | grep -E "max \||step |passed|failed|Error" | head -40
