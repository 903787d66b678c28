timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
export TPS_SHARE_DEVICE=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 4 --steps 1 --warmup 1 --model tiny --l-max 256 --prompt-len 16 --per-gpu-batch 8 --no-cpu > gpurun_out/mpbench_4.log 2>&1
echo "rc=$?"; grep -v "^tps watchdog" gpurun_out/mpbench_4.log | grep '^{' | cut -c1-600
