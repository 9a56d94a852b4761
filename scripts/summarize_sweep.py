"""Markdown table of a bench sweep (scripts/gpu_sweep_all.sh output logs)."""
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "sweep"
rows = []
for path in sorted(glob.glob(os.path.join("gpurun_out", f"{tag}_*.log"))):
    w = os.path.basename(path)[len(tag) + 1:-4]
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        rows.append(f"| {w} | failed | | | | | |")
        continue
    pc = d["roofline"]["per_class"]
    cls = " ".join(f"{k} {v['ms_per_launch']:.3f}" for k, v in pc.items())
    ps = d.get("powersgd") or {}
    rows.append(f"| {w} | {d['ms_per_step']:.3f} | {d['value']:.0f} | {d['step_hbm_frac_16B']:.2f} | "
                f"{d['roofline']['kernel']} {d['roofline']['frac']:.2f} | {cls} | "
                f"{ps.get('ms_per_step', float('nan')):.3f} ({ps.get('acp_speedup', float('nan')):.2f}x) |")
print(f"# Bench sweep `{tag}` (1x B200, 30 timed steps, CUDA graphs)\n")
print("| workload | ms/step | GB/s | 16B-floor frac | dominant kernel, roofline frac | per-class ms/launch | Power-SGD ms/step (ACP speedup) |")
print("|---|---|---|---|---|---|---|")
print("\n".join(rows))
