for v in 0 1; do TPS_ATTN_SPLIT_NKV1=$v timeout 900 python tools/solo_step.py qwen2.5-7b 8,4 12,16,24,32,48,64 3072 "" 2>&1 | grep -v watchdog | sed "s/^/split_nkv1=$v /"; done
