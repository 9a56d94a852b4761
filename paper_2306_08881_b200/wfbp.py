"""Wait-free back-propagation (WFBP) driver for a torch module (
SURVEY NEXT-2): ACP-SGD starts compressing and all-reducing a bucket as soon
as the backward pass has produced every gradient in it, overlapping the rest
of the backward pass, instead of after the whole backward pass ("naive").

The parameters are taken in READY order (reverse registration order, the
order autograd produces their gradients), the library plans the
buckets (25 MiB x compression rate per parity), and a
post-accumulate-grad hook per parameter counts the bucket down. Everything
numerical happens in the library (libacp.so) through acp_step_begin /
acp_bucket_ready / acp_step_end; this module only does bookkeeping.

    wf = Wfbp(model, rank=4, world_size=..., nccl_comm=...)
    for it in range(steps):
        wf.begin(parity=it % 2)      # zeroes .grad, orthogonalises the factors
        loss = model(...); loss.backward()
        wf.end()                     # decoded gradients are in p.grad
        opt.step()
"""
from __future__ import annotations

from typing import Optional

from .acp import AcpContext, DEFAULT_BUCKET_BYTES, verify_plan_across_ranks


class Wfbp:
    def __init__(self, model, rank: int, *, world_size: int = 1, nccl_comm: Optional[int] = None,
                 seed: int = 0, bucket_bytes: int = DEFAULT_BUCKET_BYTES, flags: int = 0,
                 overlap: bool = True, side_stream: bool = True):
        import torch
        params = [p for p in model.parameters() if p.requires_grad]
        self.params = list(reversed(params))  # ready order
        for p in self.params:  # persistent gradient storage: the library keeps the pointers
            if p.grad is None:
                p.grad = torch.zeros_like(p, memory_format=torch.contiguous_format)
        self.ctx = AcpContext([tuple(p.shape) for p in self.params], rank, world_size=world_size,
                              nccl_comm=nccl_comm, seed=seed, bucket_bytes=bucket_bytes, flags=flags)
        if world_size > 1:
            # every rank must issue the same bucket sequence; the
            # library issues its all-reduces in bucket-index order whatever
            # order the hooks fire in, but the buckets themselves must match
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized() and \
                    not verify_plan_across_ranks(self.ctx.plan()):
                raise RuntimeError("ranks derived different fused-buffer plans (different parameter lists?)")
        self.overlap = overlap
        self.bucket_of = [[int(self.ctx.plan_info(i)[4 + par]) for i in range(len(self.params))]
                          for par in (0, 1)]
        self.size = [[0] * len(self.ctx.buckets(par)) for par in (0, 1)]
        for par in (0, 1):
            for b in self.bucket_of[par]:
                self.size[par][b] += 1
        self.index = {id(p): i for i, p in enumerate(self.params)}
        self.side = torch.cuda.Stream() if side_stream else None
        self.parity = None
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]

    @property
    def grads(self):
        return [p.grad for p in self.params]

    def num_buckets(self, parity: int) -> int:
        return len(self.size[parity])

    def begin(self, parity: int) -> None:
        """Zero the gradients and open the step (orthogonalise the factors)."""
        import torch
        for p in self.params:
            p.grad.zero_()
        self.parity = parity
        self.left = list(self.size[parity])
        if not self.overlap:
            return  # naive: one whole acp_step after the backward pass
        self.ctx.step_begin(self.grads, parity)
        if self.side is not None:
            self.side.wait_stream(torch.cuda.current_stream())

    def _ready(self, b: int) -> None:
        import torch
        if self.side is not None:
            # K1 on a side stream: it overlaps the remaining backward kernels
            self.side.wait_stream(torch.cuda.current_stream())
            self.ctx.bucket_ready(b, stream=self.side)
        else:
            self.ctx.bucket_ready(b)

    def _on_grad(self, p) -> None:
        if self.parity is None or not self.overlap:
            return
        b = self.bucket_of[self.parity][self.index[id(p)]]
        self.left[b] -= 1
        if self.left[b] == 0:
            self._ready(b)

    def end(self) -> None:
        """Close the step: (naive mode) compress every bucket now, then wait
        for the all-reduces and decode into p.grad."""
        import torch
        if not self.overlap:
            self.ctx.step(self.grads, self.parity)  # the whole step (CUDA graph)
            self.parity = None
            return
        if any(self.left):
            raise RuntimeError(f"buckets without gradients: {[b for b, n in enumerate(self.left) if n]}")
        if self.side is not None:
            torch.cuda.current_stream().wait_stream(self.side)
        self.ctx.step_end()
        self.parity = None

    def close(self) -> None:
        for h in self._hooks:
            h.remove()
        self.ctx.close()
