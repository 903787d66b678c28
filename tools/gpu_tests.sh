echo "== early"; TPS_LIB_PATH=$PWD/build_variants/diag5.so TPS_ATTN_CLUSTER_EARLY=1 timeout 600 python tools/graph_probe.py 2>&1 | grep -v watchdog | sort | uniq -c | head
echo "== late"; TPS_LIB_PATH=$PWD/build_variants/diag5.so TPS_ATTN_CLUSTER_EARLY=0 timeout 600 python tools/graph_probe.py 2>&1 | grep -v watchdog | sort | uniq -c | head
