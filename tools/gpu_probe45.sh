for mc in 16 8 4; do
TPS_ATTN_MAX_CLUSTER=$mc timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,4,8,16 3072 "" 2>&1 | grep -v watchdog | sed "s/^/maxcl=$mc /"
done
