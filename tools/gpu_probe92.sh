timeout 300 python tools/qkv_probe.py 2>&1 | head -3
for v in "" build_variants/st4.so build_variants/st5.so; do
  echo "== lib $v"
  env ${v:+TPS_LIB_PATH=$PWD/$v} timeout 600 python tools/solo_step.py qwen2.5-7b 1,8 1,16,64 2048 2>&1 | grep -v watchdog
done
echo "== qkv off"
TPS_QKV_CLUSTER=0 timeout 600 python tools/solo_step.py qwen2.5-7b 1,8 1,16,64 2048 2>&1 | grep -v watchdog
