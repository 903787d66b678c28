TPS_ATTN_CLUSTER_EARLY=1 timeout 600 python tools/graph_probe.py sync 2>&1 | grep -v watchdog
