# Per-shape throughput probe: each distinct matrix shape of a model, replicated
# to ~200 MB of gradient, stepped through the library; per-class GB/s.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from acp_inputs import ready_order
from paper_2306_08881_b200 import AcpContext
model = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 4
shapes = sorted({tuple(s) for _, s in ready_order(model) if len(s) > 1}, key=lambda s: -int(torch.tensor(s).prod()))
for s in shapes:
    n = int(torch.tensor(s).prod())
    reps = max(1, int(50e6 // n))
    ctx = AcpContext([s] * reps, rank)
    g = [torch.rand(s, device="cuda") for _ in range(reps)]
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
    for k in ("proj_p", "proj_q", "decode_p", "decode_q"):
        v = pr[k]
        if v["launches"]:
            out.append(f"{k} {v['bytes'] / (v['ms'] * 1e-3) / 1e9:6.0f}")
    print(f"{str(s):22s} n*m={n:8d} x{reps:4d}  " + "  ".join(out) + " GB/s", flush=True)
    ctx.close()
    del g
    torch.cuda.empty_cache()
