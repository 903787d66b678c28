timeout 900 python -m pytest tests/test_gpu_coordinator.py tests/test_gpu_reshard_fullsize.py tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -2
timeout 300 python tools/switch_bench.py --modes 1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('switch_device_ms','host_plan_s','host_build_s','host_capture_s','copy_gbps')})"
