timeout 300 python tools/switch_bench.py --modes 0,1 2>&1 | grep -o '"copy_gbps": [0-9.]*\|"copy_launches": [0-9]*' | tr '\n' ' '; echo
