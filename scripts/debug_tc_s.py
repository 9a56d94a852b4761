# Debug helper: one P-step (ragged layer set) through the split API for two
# workers; reports per layer which (row tile, column tile) blocks of E
# disagree with the oracle.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
from acp_harness import make_inputs, make_q0, run_gpu_simulated, run_oracle
RAGGED = [(1000,), (64, 3, 7, 7), (2, 1024), (1, 8), (3, 9000), (64, 64), (256, 64), (5, 3, 2),
          (300, 1152), (17,), (130, 20), (512, 4608), (4, 4)]
rank = int(sys.argv[1]) if len(sys.argv) > 1 else 8
keep = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(len(RAGGED)))
shapes = [RAGGED[i] for i in keep]
nw = 2
inputs = make_inputs(shapes, nw, 1, 2306088, "lowrank")
q0 = make_q0(shapes, rank, 2306088)
gpu = run_gpu_simulated(shapes, rank, inputs, q0=q0, seed=2306088)
ref = run_oracle(shapes, rank, inputs, q0=q0, seed=2306088)
for li, s in enumerate(shapes):
    if len(s) == 1:
        continue
    for w in range(nw):
        E = gpu[0]["E"][w][li][2]
        R = ref[0]["E"][w][li]
        err = np.abs(E - R)
        scale = max(np.abs(R).max(), 1e-30)
        bad = err > 1e-3 * scale
        if bad.any():
            rows = np.where(bad.any(axis=1))[0]
            cols = np.where(bad.any(axis=0))[0]
            print(s, "worker", w, "bad", int(bad.sum()), "of", bad.size, "rows", rows.min(), rows.max(),
                  "cols", cols.min(), cols.max(), "row tiles", sorted(set((rows // 128).tolist())),
                  "col tiles", sorted(set((cols // 64).tolist()))[:20])
print("done")
