timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 1 0; do
TPS_NORM_CLUSTER=$c timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,8 1,16,64 2048 "" 2>&1 | grep -v watchdog | sed "s/^/cluster=$c /"
done
