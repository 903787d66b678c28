timeout 900 python -m pytest tests/test_gpu_coordinator.py tests/test_gpu_reshard_fullsize.py tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -2
