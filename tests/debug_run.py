"""Tiny end-to-end run of every kernel class (debug builds with device-side
checks, ACP_LIB=...): K2 (CholeskyQR2), the SIMT stream K1 / decode
kernels (r = 4, deferred residual; 1-D packing; the generic path), the
tensor-core kernels (r = 8: K1 P/Q steps, column reduce, decodes), the
register row/column kernels (NO_EF), state access, for a few alternating
steps, eagerly and through a captured graph. Prints 'debug run ok'."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_08881_b200 import AcpContext, ACP_NO_EF  # noqa: E402


def main():
    torch.cuda.set_device(0)
    shapes = [(40,), (96, 1024), (33, 147), (64, 256), (7, 3, 3), (130, 20), (24, 4096)]
    g0 = torch.Generator(device="cuda").manual_seed(0)
    for rank, flags in ((4, 0), (8, 0), (2, ACP_NO_EF)):
        for graphs in (False, True):
            ctx = AcpContext(shapes, rank, seed=3, flags=flags)
            ctx.set_graphs(graphs)
            for t in range(4):
                g = [torch.randn(s, device="cuda", generator=g0) for s in shapes]
                ctx.step(g, t % 2)
            P, Q, E = ctx.get_state(1)
            ctx.set_state(1, P, Q, E)
            ctx.step(g, 0)
            torch.cuda.synchronize()
            ctx.close()
    print("debug run ok")


if __name__ == "__main__":
    main()
