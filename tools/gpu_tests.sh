timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/graph_probe.py 2>&1 | grep -v watchdog
