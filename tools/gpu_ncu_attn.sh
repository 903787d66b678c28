NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_attn_kernel --launch-skip 60 -c 1 -o gpurun_out/ncu_attn_split_b64 -f python tools/solo_once.py qwen2.5-7b 1 64 1024 2 > /dev/null 2>&1
ls -la gpurun_out/ncu_attn_split_b64.ncu-rep
