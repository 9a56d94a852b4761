# K2 (orth) time per launch for one replicated shape: P-steps orthogonalise the
# m-side factors, Q-steps the n-side; prints us per launch for each parity.
# usage: python scripts/k2_probe.py ROWS COLS COUNT RANK
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2306_08881_b200 import AcpContext
n, m, cnt, rank = (int(x) for x in sys.argv[1:5])
ctx = AcpContext([(n, m)] * cnt, rank)
g = [torch.rand((n, m), device="cuda") for _ in range(cnt)]
for t in range(4):
    ctx.step(g, t % 2)
res = []
for par in (0, 1):
    ctx.profile(True)
    ctx.profile_reset()
    for t in range(6):
        ctx.step(g, par if t % 2 == 0 else 1 - par)
    torch.cuda.synchronize()
    pr = ctx.profile_read()
    ctx.profile(False)
    res.append(pr["orth"]["ms"] / max(1, pr["orth"]["launches"]) * 1e3)
print(f"{n}x{m} x{cnt} r={rank}: K2 avg us/launch {sum(res)/2:.1f}", flush=True)
ctx.close()
