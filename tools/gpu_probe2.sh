# stage breakdown + step sweeps + ncu full captures of the top kernels
mkdir -p gpurun_out
timeout 600 python tools/stage_breakdown.py --out gpurun_out/stage_breakdown.json > gpurun_out/stage_breakdown.log 2>&1
for ctx in 512 2048 8192; do
  timeout 300 python tools/quick_step.py qwen2.5-7b 1,2,4,8,16,32,64 $ctx >> gpurun_out/quick_step.log 2>&1
done
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_swapab --launch-skip 400 -c 2 \
  -o gpurun_out/ncu_gemm_b64 -f python tools/quick_step.py qwen2.5-7b 64 2048 > gpurun_out/ncu_gemm_b64.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_swapab --launch-skip 400 -c 2 \
  -o gpurun_out/ncu_gemm_b1 -f python tools/quick_step.py qwen2.5-7b 1 2048 > gpurun_out/ncu_gemm_b1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_attn --launch-skip 100 -c 2 \
  -o gpurun_out/ncu_attn_b64 -f python tools/quick_step.py qwen2.5-7b 64 4096 > gpurun_out/ncu_attn_b64.log 2>&1
ls -la gpurun_out
