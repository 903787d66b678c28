mkdir -p gpurun_out
free -g | head -2; nproc
timeout 2400 python -m pytest tests/test_gpu_decode_fullshape.py -q -s -k "full_depth or wide_batch" --durations=20 > gpurun_out/pytest_fullshape.log 2>&1; tail -40 gpurun_out/pytest_fullshape.log
