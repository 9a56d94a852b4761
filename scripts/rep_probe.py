# Whole-model replication probe: the model's layer set repeated k times.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from acp_inputs import ready_order
from paper_2306_08881_b200 import AcpContext
model = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 4
base = [tuple(s) for _, s in ready_order(model)]
for k in (1, 2, 4, 8):
    shapes = base * k
    n = sum(int(torch.tensor(s).prod()) for s in shapes)
    ctx = AcpContext(shapes, rank)
    g = [torch.rand(s, device="cuda") for s in shapes]
    for t in range(4):
        ctx.step(g, t % 2)
    ctx.profile(True)
    ctx.profile_reset()
    for t in range(6):
        ctx.step(g, t % 2)
    torch.cuda.synchronize()
    pr = ctx.profile_read()
    ctx.profile(False)
    out = []
    for c in ("orth", "proj_p", "proj_q", "decode_p", "decode_q"):
        v = pr[c]
        if v["launches"]:
            out.append(f"{c} {v['ms'] / v['launches'] * 1e3:7.1f}us {v['bytes'] / (v['ms'] * 1e-3) / 1e9:5.0f}GB/s")
    print(f"x{k} elements {n/1e6:6.1f}M  " + "  ".join(out), flush=True)
    ctx.close()
    del g
    torch.cuda.empty_cache()
