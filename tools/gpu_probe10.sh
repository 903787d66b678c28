for c in 0 1; do
TPS_CARVEOUT=$c timeout 600 python tools/solo_step.py qwen2.5-7b 1,8 1,64 2048 ";attention,qkv_rope,add_norm;linear" 2>&1 | sed "s/^/carveout=$c /" | grep -v watchdog
done
