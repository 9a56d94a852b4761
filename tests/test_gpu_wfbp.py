"""WFBP driver (paper_2306_08881_b200/wfbp.py, acp_step_begin / acp_bucket_ready
/ acp_step_end): the bucket-granular step driven
by autograd hooks gives the same decoded gradients as acp_step on the same
raw gradients (different CTA splits: equal to fp32 rounding)."""
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


def _model(seed):
    import torch
    torch.manual_seed(seed)
    return torch.nn.Sequential(
        torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.LayerNorm(512),
        torch.nn.Linear(512, 512), torch.nn.ReLU(), torch.nn.Linear(512, 1000)).cuda()


@pytest.mark.parametrize("overlap,bucket_bytes", [(True, 25 * 2 ** 20), (True, 0), (False, 25 * 2 ** 20)])
def test_wfbp_matches_step(overlap, bucket_bytes):
    import torch
    from paper_2306_08881_b200 import AcpContext
    from paper_2306_08881_b200.wfbp import Wfbp
    model = _model(0)
    ref_model = _model(0)
    wf = Wfbp(model, 4, seed=5, bucket_bytes=bucket_bytes, overlap=overlap)
    ready = list(reversed([p for p in ref_model.parameters()]))
    ctx = AcpContext([tuple(p.shape) for p in ready], 4, seed=5, bucket_bytes=bucket_bytes)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for t in range(4):
        x = torch.randn(64, 256, device="cuda", generator=gen)
        wf.begin(t % 2)
        model(x).square().mean().backward()
        wf.end()
        for p in ref_model.parameters():
            p.grad = None
        ref_model(x).square().mean().backward()
        g = [p.grad.contiguous() for p in ready]
        ctx.step(g, t % 2)
        torch.cuda.synchronize()
        for a, b in zip(wf.grads, g):
            err = (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b).clamp_min(1e-30)).item()
            assert err <= 1e-5, (t, err)
    wf.close()
    ctx.close()


def test_bucket_api_errors():
    import torch
    from paper_2306_08881_b200 import AcpContext, AcpError
    shapes = [(64, 64), (64,), (128, 32)]
    ctx = AcpContext(shapes, 4, bucket_bytes=0)
    g = [torch.randn(s, device="cuda") for s in shapes]
    with pytest.raises(AcpError):
        ctx.bucket_ready(0)          # no open step
    ctx.step_begin(g, 0)
    with pytest.raises(AcpError):
        ctx.step_begin(g, 0)         # already open
    ctx.bucket_ready(0)
    with pytest.raises(AcpError):
        ctx.bucket_ready(0)          # twice
    with pytest.raises(AcpError):
        ctx.bucket_ready(99)         # out of range
    with pytest.raises(AcpError):
        ctx.step_end()               # buckets missing
    for b in range(1, len(ctx.buckets(0))):
        ctx.bucket_ready(b)
    ctx.step_end()
    torch.cuda.synchronize()
    ctx.close()
