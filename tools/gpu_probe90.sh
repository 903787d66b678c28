timeout 300 python tools/qkv_probe.py
TPS_QKV_CLUSTER=16 timeout 300 python tools/qkv_probe.py
