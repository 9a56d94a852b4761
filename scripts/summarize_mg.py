#!/usr/bin/env python
"""Summarise scripts/gpu_multi_r02.sh logs (profiles/r02_mgN/) into a markdown table."""
import glob
import json
import os
import sys

d = sys.argv[1]
N = sys.argv[2]
out = [f"# Round-2 multi-GPU evidence, {N}x B200 (one box, NVSwitch)", "",
       f"Raw logs: `{d}/` (`mg_parity_{N}.log` = tests/mgpu_check.py output, the bench JSON lines, `nvidia-smi topo -m`).",
       "Produced by `scripts/gpu_multi_r02.sh {N}` under `gpurun --gpus {N}`; `ms` is max over ranks, CUDA events.", ""]
par = open(os.path.join(d, f"mg_parity_{N}.log")).read().splitlines()
out += ["## Parity (tests/mgpu_check.py)", "", "```"] + [l for l in par if l.startswith("run") or "mgpu ok" in l] + ["```", ""]


def row(path):
    j = json.loads(open(path).read().strip().splitlines()[-1])
    ss = j.get("ssgd") or {}
    return j, ss


out += ["## Bench lines", "", "| workload | all-reduce | ms/step | P-step / Q-step ms | buckets P/Q | box GB/s | S-SGD ms (25 MiB NCCL) |",
        "|---|---|---|---|---|---|---|"]
for w in ("bert-large-r4", "resnet50-r4", "bert-large-r32"):
    for ar in ("nccl", "nvls"):
        p = os.path.join(d, f"mg_bench_{N}_{w}_{ar}.log")
        if not os.path.exists(p):
            continue
        j, ss = row(p)
        out.append(f"| {w} | {ar} | {j['ms_per_step']:.4f} | {j['step_stats']['p_step_ms']:.4f} / {j['step_stats']['q_step_ms']:.4f} "
                   f"| {j['config'].get('buckets_PQ')} | {j['value']:.0f} | {ss.get('ms_per_step', '')} |")
out += ["", "## ResNet-152 r=4 tensor-fusion buffer sweep (BASELINE configs[2]; P:342-357)", "",
        "`default_bucket_bytes` scaled by the per-parity compression rate (P:257); 0 = one tensor per bucket, -1 = one bucket.", "",
        "| bucket bytes | buckets P/Q | NCCL ms/step | NVLS (fused into the decode) ms/step |", "|---|---|---|---|"]
for bb in ("0", "1048576", "5242880", "26214400", "104857600", "-1"):
    a = os.path.join(d, f"mg_sweep_{N}_{bb}_nccl.log")
    b = os.path.join(d, f"mg_sweep_{N}_{bb}_nvls.log")
    if not (os.path.exists(a) and os.path.exists(b)):
        continue
    ja, _ = row(a)
    jb, _ = row(b)
    lab = {"0": "0 (per tensor)", "-1": "single"}.get(bb, f"{int(bb) // 2 ** 20} MiB")
    out.append(f"| {lab} | {ja['config'].get('buckets_PQ')} | {ja['ms_per_step']:.4f} | {jb['ms_per_step']:.4f} |")
print("\n".join(out))
