for cfg in "32 2 3" "16 2 6" "16 3 4" "24 2 4" "48 2 2" "16 2 4" "32 2 3"; do
  set -- $cfg
  echo "== buf ${1}KB depth $2 ctas/SM $3"
  TPS_COPY_BUF_KB=$1 TPS_COPY_DEPTH=$2 TPS_COPY_CTAS_PER_SM=$3 timeout 300 python tools/switch_bench.py --modes 1 2>&1 | grep -o '"copy_gbps": [0-9.]*\|"copy_kernel_ms": [0-9.]*' | tr '\n' ' '; echo
done
