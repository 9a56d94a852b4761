# Minimal reproduction helper: ragged layer set through the split API at one rank.
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from acp_harness import make_inputs, make_q0, run_gpu_simulated, run_oracle, compare
RAGGED = [(1000,), (64, 3, 7, 7), (2, 1024), (1, 8), (3, 9000), (64, 64), (256, 64), (5, 3, 2),
          (300, 1152), (17,), (130, 20), (512, 4608), (4, 4)]
rank = int(sys.argv[1]) if len(sys.argv) > 1 else 32
only = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else None
shapes = [RAGGED[i] for i in only] if only else RAGGED
inputs = make_inputs(shapes, 2, 3, 2306088, "lowrank")
q0 = make_q0(shapes, rank, 2306088)
gpu = run_gpu_simulated(shapes, rank, inputs, q0=q0, seed=2306088)
ref = run_oracle(shapes, rank, inputs, q0=q0, seed=2306088)
print(compare(shapes, gpu, ref, inputs))
