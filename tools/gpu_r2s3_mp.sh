mkdir -p gpurun_out/mp
run() { tag=$1; dir=$2; shift; shift; (cd $dir && env "$@" TPS_SHARE_DEVICE=1 OMP_NUM_THREADS=1 timeout 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tests/mp_stage_worker.py /tmp tiny "" > $GRAFT_REPO_ROOT/gpurun_out/mp/log_$tag.txt 2>&1); echo "$tag rc=$? $(grep -c watchdog gpurun_out/mp/log_$tag.txt)"; }
for i in 1 2 3 4 5 6; do run new$i . X=1; done
timeout 300 python -m pytest -x -q tests/test_gpu_kernels.py -k barrier 2>&1 | tail -2
