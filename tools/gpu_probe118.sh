TPS_LIB_PATH=$PWD/build_variants/diag2.so TPS_ATTN_CLUSTER_EARLY=1 timeout 600 python tools/graph_probe.py 2>&1 | grep -v watchdog
