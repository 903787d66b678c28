timeout 900 python tools/graph_probe.py wide 2>&1 | grep -v watchdog
timeout 600 python tools/graph_probe.py 2>&1 | grep -v watchdog
