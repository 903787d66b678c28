mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_persist.py -x -q -s 2>&1 | tail -30 > gpurun_out/persist_tests.log; cat gpurun_out/persist_tests.log
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -5
