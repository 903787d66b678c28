mkdir -p gpurun_out
export TPS_SHARE_DEVICE=1
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps 1 --warmup 1 --model tiny --l-max 256 --prompt-len 16 --per-gpu-batch 8 --no-cpu > gpurun_out/mpbench_$n.log 2>&1
tail -c 2500 gpurun_out/mpbench_$n.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --model tiny --l-max 256 --prompt-len 16 --per-gpu-batch 8 > gpurun_out/mpbench_ref.log 2>&1
tail -c 1500 gpurun_out/mpbench_ref.log
