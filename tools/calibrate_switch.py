"""Derive the Switch Executor constants of presets/b200.cfg from the measured config-5 sweep.

python tools/calibrate_switch.py profiles/r2/switch_sweep_qwen7b.jsonl [...]

  t_fixed_control : median of (switch device time - copy-kernel time): barriers, the expander,
                    launch gaps and host work left on the critical path (virtual world: no
                    NVLink barrier latency; the multi-process barrier adds ~10-20 us)
  copy efficiency : copy-kernel bytes / time vs the HBM copy peak (read + write) -- applied to
                    the 770 GB/s measured NVLink peer copy for intra_bw_unidir
  graph / comm    : host seconds of graph capture and layout build inside a switch
"""
import json, statistics, sys

rows = [json.loads(l) for p in sys.argv[1:] for l in open(p) if l.startswith("{")]
ok = [r for r in rows if "copy_kernel_ms" in r]
fixed = [r["switch_device_ms"] - r["copy_kernel_ms"] for r in ok]
eff = [2 * r["copy_gbps"] / 6547.8 for r in ok]
big = [2 * r["copy_gbps"] / 6547.8 for r in ok if r["copy_bytes"] / max(1, r["copy_launches"]) > 2e9]
out = {
    "points": len(ok), "skipped": len(rows) - len(ok),
    "t_fixed_control_ms": {"median": statistics.median(fixed), "p90": sorted(fixed)[int(0.9 * len(fixed))],
                           "max": max(fixed)},
    "copy_efficiency_vs_hbm_copy_peak": {"median": statistics.median(eff), "min": min(eff), "max": max(eff),
                                         "large_items_median": statistics.median(big) if big else None},
    "graph_capture_in_switch_s": max(r["host_capture_s"] for r in ok),
    "layout_build_in_switch_s": max(r["host_build_s"] for r in ok),
    "device_over_copy": {"median": statistics.median(r["switch_device_ms"] / r["copy_kernel_ms"] for r in ok),
                         "max": max(r["switch_device_ms"] / r["copy_kernel_ms"] for r in ok)},
}
out["intra_bw_unidir"] = 770e9 * out["copy_efficiency_vs_hbm_copy_peak"]["median"]
print(json.dumps(out, indent=1))
