timeout 600 python tools/solo_step.py qwen2.5-7b 2,4,8 1,16,64 2048 ";fuse_push;attention,qkv_rope,add_norm;linear" > gpurun_out/solo_step.log 2>&1
grep -v watchdog gpurun_out/solo_step.log | head -60
