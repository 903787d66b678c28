# one-process-per-rank bench path with the real Qwen2.5-7B geometry, both ranks on cuda:0
mkdir -p gpurun_out
export TPS_SHARE_DEVICE=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
  bench.py --gpus 2 --steps 1 --warmup 1 --per-gpu-batch 8 --l-max 512 --prompt-len 128 --no-cpu --no-e2e \
  > gpurun_out/mpbench_qwen2.log 2>&1
echo "rc=$?"
grep -v "^tps watchdog" gpurun_out/mpbench_qwen2.log | tail -c 2500
