"""Determinism probe: run the same seeded steps several times through the
library and compare every tensor's decoded gradient and state bitwise across
runs (the kernels are deterministic by construction, so any difference is a
race). usage: python scripts/race_probe.py MODEL RANK [REPS] [STEPS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from acp_inputs import gradient_for_shape, ready_order  # noqa: E402
from acp_harness import make_q0  # noqa: E402
from paper_2306_08881_b200 import AcpContext  # noqa: E402


def run(shapes, rank, steps, host):
    q0 = make_q0(shapes, rank, 7)
    ctx = AcpContext(shapes, rank, seed=7, q0=q0)
    ctx.set_graphs(True)
    outs = []
    for t in range(steps):
        grads = [torch.from_numpy(h).cuda() for h in host[t]]
        ctx.step(grads, t % 2)
        torch.cuda.synchronize()
        dec = [g.cpu().numpy() for g in grads]
        st = []
        for i, s in enumerate(shapes):
            if len(s) > 1:
                P, Q, E = ctx.get_state(i)
                st.append((P.cpu().numpy(), Q.cpu().numpy(), E.cpu().numpy()))
            else:
                st.append(None)
        outs.append((dec, st))
    ctx.close()
    return outs


def main():
    model, rank = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    shapes = [s for _, s in ready_order(model)]
    host = [[np.ascontiguousarray(gradient_for_shape(s, seed=7, worker=0, layer=i, step=t))
             for i, s in enumerate(shapes)] for t in range(steps)]
    base = run(shapes, rank, steps, host)
    bad = 0
    for rep in range(1, reps):
        o = run(shapes, rank, steps, host)
        for t in range(steps):
            for i, s in enumerate(shapes):
                if not np.array_equal(o[t][0][i], base[t][0][i]):
                    d = np.abs(o[t][0][i] - base[t][0][i])
                    print(f"rep {rep} step {t} tensor {i} {s}: decoded differs, max {d.max():.3e}")
                    bad += 1
                if o[t][1][i] is not None:
                    for nm, a, b in zip("PQE", o[t][1][i], base[t][1][i]):
                        if not np.array_equal(a, b):
                            dd = np.abs(a - b)
                            rows = np.unique(np.nonzero(dd.reshape(dd.shape[0], -1) if nm != 'E' else dd.reshape(s[0], -1))[0])
                            print(f"rep {rep} step {t} tensor {i} {s}: {nm} differs, max {dd.max():.3e}, rows {rows[:12]} ({len(rows)})")
                            bad += 1
    print(f"{model} r={rank}: {bad} differences over {reps} runs x {steps} steps")


if __name__ == "__main__":
    main()
