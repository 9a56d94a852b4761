"""CPU oracle for ACP-SGD / Power-SGD -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package. The CUDA path
(``paper_2306_08881_b200``) never imports it and shares no code with it; the
two meet only through seeded inputs from ``acp_inputs``.

Pinned by tests/test_oracle_*.py against what PAPER.md and mathematics fix
(closed forms, the paper's printed numbers, invariants, brute force).
Parity unpinned: the full multi-step trajectory of decoded gradients and
errors on generic inputs is pinned only through the invariants (see
DESIGN.md "Parity pins").
"""
from .acp_oracle import (AcpOracle, PowerSgdOracle, DegenerateFactor,  # noqa: F401
                         orthogonalize, reshape_policy, layer_rank, make_layers,
                         reference_reduce, payload_elems, compression_rates,
                         buffer_cap_bytes, plan_buckets, fusion_plan, rel_frobenius,
                         DEFAULT_BUCKET_BYTES)
from . import rng  # noqa: F401
