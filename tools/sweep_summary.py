"""Markdown summary of a config-5 switch sweep (tools/switch_bench.py JSON lines)."""
import json, sys

rows = [json.loads(l) for p in sys.argv[1:] for l in open(p) if l.startswith("{")]
print("| model | world | tp | samples x ctx | weights GB | KV GB | max GPU peer GB | max GPU local GB | copy ms | "
      "switch ms | switch/copy | copy GB/s (r+w frac of 6548) | NVLink floor ms* |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    if "copy_kernel_ms" not in r:
        print(f"| {r['model']} | {r['world']} | {r['tp']} | {r['samples']} x {r['ctx']} | skipped: {r['skipped']} |"
              " | | | | | | | |")
        continue
    floor = r["max_gpu_peer_bytes"] / 770e9 * 1e3
    print(f"| {r['model']} | {r['world']} | {r['tp']} | {r['samples']} x {r['ctx']} | {r['weights_bytes']/1e9:.2f} | "
          f"{r['kv_bytes']/1e9:.2f} | {r['max_gpu_peer_bytes']/1e9:.2f} | {r['max_gpu_local_bytes']/1e9:.2f} | "
          f"{r['copy_kernel_ms']:.2f} | {r['switch_device_ms']:.2f} | {r['switch_device_ms']/r['copy_kernel_ms']:.2f} | "
          f"{r['copy_gbps']:.0f} ({2*r['copy_gbps']/6547.8:.2f}) | {floor:.2f} |")
print("\n*max per-GPU peer bytes at the measured 770 GB/s NVLink peer copy: what the same switch needs on an 8xB200 "
      "node at least (here every rank shares one GPU, so every byte is an HBM copy).")
