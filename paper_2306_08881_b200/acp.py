"""Python face of the C ABI: ``AcpContext`` (one data-parallel worker).

PyTorch provides the device memory (workspace, gradients), the CUDA stream and
the process group used to bootstrap NCCL; every step of the hot path runs in
the library's sm_100a kernels and NCCL.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

DEFAULT_BUCKET_BYTES = 25 * 2 ** 20


def _shape_rows_cols(shapes):
    rows, cols = [], []
    for s in shapes:
        s = tuple(int(d) for d in s)
        if len(s) == 0:
            raise ValueError("scalar tensors are not supported")
        if len(s) == 1:
            rows.append(s[0]); cols.append(0)            # vector: uncompressed
        else:
            rows.append(s[0]); cols.append(int(np.prod(s[1:])))  # n = dim0, m = prod(rest)
    return rows, cols


def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def broadcast_unique_id(uid: bytes, group=None) -> bytes:
    """Broadcast group-rank 0's 128-byte NCCL unique id over ``group`` (any
    torch.distributed backend); every rank returns rank 0's bytes."""
    import torch.distributed as dist
    if len(uid) != 128:
        raise ValueError("an ncclUniqueId is 128 bytes")
    payload = [bytes(uid)]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(payload, src=src, group=group)
    return payload[0]


def nccl_comm_from_group(group=None, device: Optional[int] = None) -> int:
    """Create an NCCL communicator spanning ``group`` (torch.distributed):
    rank 0 draws the unique id, the group broadcasts it, every rank inits."""
    import torch
    import torch.distributed as dist
    lib = L.load()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        L.check(lib.acp_nccl_unique_id(uid))
    uid = (C.c_uint8 * 128).from_buffer_copy(broadcast_unique_id(bytes(uid), group))
    dev = torch.cuda.current_device() if device is None else device
    comm = C.c_void_p()
    L.check(lib.acp_nccl_comm_create(uid, world, rank, dev, C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    L.check(L.load().acp_nccl_comm_destroy(C.c_void_p(comm)))


def nccl_comm_single(device: Optional[int] = None) -> int:
    """A 1-rank NCCL communicator on this process's GPU (no process group
    needed): with ``ACP_BUCKETED`` it drives the per-bucket all-reduce path on
    one GPU."""
    import torch
    lib = L.load()
    uid = (C.c_uint8 * 128)()
    L.check(lib.acp_nccl_unique_id(uid))
    dev = torch.cuda.current_device() if device is None else device
    comm = C.c_void_p()
    L.check(lib.acp_nccl_comm_create(uid, 1, 0, dev, C.byref(comm)))
    return comm.value


def _make_config(shapes, rank, world_size, nccl_comm, seed, bucket_bytes, flags, device):
    """acp_config for parameter shapes in ready order; returns (cfg, keep)
    where keep holds the ctypes arrays the config points to."""
    rows, cols = _shape_rows_cols(shapes)
    T = len(rows)
    crow = (C.c_int64 * T)(*rows)
    ccol = (C.c_int64 * T)(*cols)
    cfg = L.AcpConfig()
    cfg.abi_version = L.ACP_ABI_VERSION
    cfg.num_tensors = T
    cfg.rows = C.cast(crow, C.POINTER(C.c_int64))
    cfg.cols = C.cast(ccol, C.POINTER(C.c_int64))
    cfg.rank = int(rank)
    cfg.world_size = int(world_size)
    cfg.nccl_comm = C.c_void_p(nccl_comm) if nccl_comm else None
    cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    cfg.default_bucket_bytes = int(bucket_bytes)
    cfg.flags = int(flags)
    cfg.device = int(device)
    return cfg, (crow, ccol)


def plan_host(shapes: Sequence[Sequence[int]], rank: int, *, world_size: int = 1,
              bucket_bytes: int = DEFAULT_BUCKET_BYTES, flags: int = 0) -> dict:
    """The library's fused-buffer plan, built on the host with no GPU
    (acp_plan_create): per tensor (r_i, P-slot, Q-slot, E offset, P-bucket,
    Q-bucket) and every bucket's [offset, count) per parity."""
    lib = L.load()
    cfg, keep = _make_config([tuple(int(d) for d in s) for s in shapes], rank, world_size, None, 0,
                             bucket_bytes, flags, -1)
    ctx = C.c_void_p()
    L.check(lib.acp_plan_create(C.byref(cfg), C.byref(ctx)))
    try:
        out = (C.c_int64 * 6)()
        tensors = []
        for i in range(len(shapes)):
            L.check(lib.acp_plan_info(ctx, i, out))
            tensors.append(tuple(int(x) for x in out))
        buckets = []
        for parity in (0, 1):
            nb = C.c_int32()
            L.check(lib.acp_num_buckets(ctx, parity, C.byref(nb)))
            rng = []
            for b in range(nb.value):
                off, cnt = C.c_int64(), C.c_int64()
                L.check(lib.acp_bucket_range(ctx, parity, b, C.byref(off), C.byref(cnt)))
                rng.append((off.value, cnt.value))
            buckets.append(rng)
    finally:
        lib.acp_destroy(ctx)
    del keep
    return {"tensors": tensors, "buckets": buckets}


class AcpContext:
    """ACP-SGD state of one worker for a list of parameter shapes in READY
    order (the order gradients become ready in back-propagation)."""

    def __init__(self, shapes: Sequence[Sequence[int]], rank: int, *, world_size: int = 1,
                 nccl_comm: Optional[int] = None, seed: int = 0,
                 q0: Optional[List[Optional[np.ndarray]]] = None,
                 bucket_bytes: int = DEFAULT_BUCKET_BYTES, flags: int = 0,
                 device=None):
        import torch
        self._lib = L.load()
        self.shapes = [tuple(int(d) for d in s) for s in shapes]
        self.rank = int(rank)
        self.world_size = int(world_size)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        T = len(self.shapes)
        cfg, self._keep = _make_config(self.shapes, self.rank, self.world_size, nccl_comm, seed,
                                       bucket_bytes, flags,
                                       dev.index if dev.index is not None else torch.cuda.current_device())
        q0buf = None
        if q0 is not None:
            parts = []
            for s, q in zip(self.shapes, q0):
                if len(s) == 1:
                    continue
                parts.append(np.ascontiguousarray(q, dtype=np.float32).ravel())
            flat = np.concatenate(parts) if parts else np.zeros(1, np.float32)
            q0buf = (C.c_float * flat.size).from_buffer_copy(flat.tobytes())
            cfg.q0_host = C.cast(q0buf, C.POINTER(C.c_float))
        nbytes = C.c_size_t()
        L.check(self._lib.acp_workspace_bytes(C.byref(cfg), C.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device=dev)
        cfg.workspace = C.c_void_p(self.workspace.data_ptr())
        cfg.workspace_bytes = nbytes.value
        ctx = C.c_void_p()
        L.check(self._lib.acp_create(C.byref(cfg), C.byref(ctx)))
        self._ctx = ctx
        self._cfg = cfg
        self._ptrs = (C.c_void_p * T)()

    # -- helpers --------------------------------------------------------------
    def _grad_ptrs(self, grads):
        """Pointer array for the C call. Tensors are validated only when the
        pointer set changes (the per-step cost is one data_ptr() per tensor)."""
        import torch
        if len(grads) != len(self.shapes):
            raise ValueError(f"expected {len(self.shapes)} gradients, got {len(grads)}")
        ptrs = [g.data_ptr() for g in grads]
        if ptrs != getattr(self, "_last_ptrs", None):
            for i, (g, s) in enumerate(zip(grads, self.shapes)):
                if not (isinstance(g, torch.Tensor) and g.is_cuda and g.dtype == torch.float32
                        and g.is_contiguous() and g.numel() == int(np.prod(s))):
                    raise ValueError(f"gradient {i} must be a contiguous fp32 CUDA tensor of shape {s}")
                self._ptrs[i] = ptrs[i]
            self._last_ptrs = ptrs
        return C.cast(self._ptrs, C.POINTER(C.c_void_p))

    # -- hot path -------------------------------------------------------------
    def step(self, grads, parity: int, stream=None) -> None:
        """One ACP-SGD step; grads are overwritten with the decoded mean."""
        L.check(self._lib.acp_step(self._ctx, int(parity), self._grad_ptrs(grads),
                                   C.c_void_p(_stream_handle(stream))))

    # -- NVLS all-reduce (acp_attach_symmetric) ------------------------------
    def attach_symmetric(self, group=None) -> bool:
        """Move the fused buffers into torch symmetric memory bound to an NVLS
        multicast object and all-reduce with the library's in-switch kernel
        instead of NCCL (collective over `group`). Returns False (nothing
        changed) when the device has no multicast support."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        if group is None:
            group = dist.group.WORLD
        need = C.c_int64()
        L.check(self._lib.acp_symmetric_bytes(self._ctx, C.byref(need)))
        buf = symm_mem.empty(int(need.value), dtype=torch.uint8, device=self.device)
        h = symm_mem.rendezvous(buf, group.group_name)
        ok = torch.tensor([1 if h.multicast_ptr else 0], device=self.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if not int(ok.item()):
            return False
        peers = (C.c_void_p * h.world_size)(*h.buffer_ptrs)
        L.check(self._lib.acp_attach_symmetric(self._ctx, C.c_void_p(buf.data_ptr()),
                                               C.c_void_p(h.multicast_ptr),
                                               C.cast(peers, C.POINTER(C.c_void_p)),
                                               int(h.rank), int(need.value)))
        torch.cuda.synchronize()
        dist.barrier(group=group)
        self._symm = (buf, h)  # keep the region alive with the context
        return True

    # -- bucket-granular step (WFBP, acp_step_begin / acp_bucket_ready / acp_step_end)
    def step_begin(self, grads, parity: int, stream=None) -> None:
        """Open a step: orthogonalise the reused factors. The gradient tensors
        must keep their storage until step_end."""
        L.check(self._lib.acp_step_begin(self._ctx, int(parity), self._grad_ptrs(grads),
                                         C.c_void_p(_stream_handle(stream))))

    def bucket_ready(self, bucket: int, stream=None) -> None:
        """All tensors of `bucket` (this parity's bucket, ready order) hold their
        gradients: project + pack them and start the bucket's all-reduce."""
        L.check(self._lib.acp_bucket_ready(self._ctx, int(bucket), C.c_void_p(_stream_handle(stream))))

    def step_end(self, stream=None) -> None:
        """Wait for every bucket's all-reduce and decode into the gradients."""
        L.check(self._lib.acp_step_end(self._ctx, C.c_void_p(_stream_handle(stream))))

    def compress(self, grads, parity: int, stream=None):
        """Split API: returns the parity's fused buffer as a torch view."""
        import torch
        buf = C.c_void_p()
        cnt = C.c_int64()
        L.check(self._lib.acp_compress(self._ctx, int(parity), self._grad_ptrs(grads),
                                       C.byref(buf), C.byref(cnt),
                                       C.c_void_p(_stream_handle(stream))))
        # the buffer lives in the workspace, or (after attach_symmetric) in
        # the symmetric region: view whichever allocation holds it
        holder = self._symm[0] if getattr(self, "_symm", None) else self.workspace
        off = buf.value - holder.data_ptr()
        if off < 0 or off + 4 * cnt.value > holder.numel():
            raise RuntimeError("acp_compress returned a buffer outside the context's allocations")
        return holder[off:off + 4 * cnt.value].view(torch.float32)

    def decompress(self, grads, parity: int, stream=None) -> None:
        L.check(self._lib.acp_decompress(self._ctx, int(parity), self._grad_ptrs(grads),
                                         C.c_void_p(_stream_handle(stream))))

    # -- state / plan ---------------------------------------------------------
    def get_state(self, i: int, stream=None):
        import torch
        n, m = self.shapes[i][0], int(np.prod(self.shapes[i][1:]))
        r = self.plan_info(i)[0]
        P = torch.empty((n, r), dtype=torch.float32, device=self.device)
        Q = torch.empty((m, r), dtype=torch.float32, device=self.device)
        E = torch.empty((n, m), dtype=torch.float32, device=self.device)
        L.check(self._lib.acp_get_state(self._ctx, i, C.c_void_p(P.data_ptr()),
                                        C.c_void_p(Q.data_ptr()), C.c_void_p(E.data_ptr()),
                                        C.c_void_p(_stream_handle(stream))))
        return P, Q, E

    def set_state(self, i: int, P=None, Q=None, E=None, stream=None) -> None:
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
        L.check(self._lib.acp_set_state(self._ctx, i, ptr(P), ptr(Q), ptr(E),
                                        C.c_void_p(_stream_handle(stream))))

    def plan_info(self, i: int) -> Tuple[int, int, int, int, int, int]:
        out = (C.c_int64 * 6)()
        L.check(self._lib.acp_plan_info(self._ctx, i, out))
        return tuple(int(x) for x in out)

    def plan(self) -> dict:
        """Same structure as ``plan_host`` (for verify_plan_across_ranks)."""
        return {"tensors": [self.plan_info(i) for i in range(len(self.shapes))],
                "buckets": [self.buckets(0), self.buckets(1)]}

    def buckets(self, parity: int) -> List[Tuple[int, int]]:
        nb = C.c_int32()
        L.check(self._lib.acp_num_buckets(self._ctx, parity, C.byref(nb)))
        res = []
        for b in range(nb.value):
            off, cnt = C.c_int64(), C.c_int64()
            L.check(self._lib.acp_bucket_range(self._ctx, parity, b, C.byref(off), C.byref(cnt)))
            res.append((off.value, cnt.value))
        return res

    # -- profiling ------------------------------------------------------------
    def profile(self, enable: bool = True) -> None:
        L.check(self._lib.acp_profile_enable(self._ctx, 1 if enable else 0))

    def profile_reset(self) -> None:
        L.check(self._lib.acp_profile_reset(self._ctx))

    def profile_read(self) -> dict:
        out = {}
        for k, name in enumerate(L.KERNEL_CLASS_NAMES):
            ms, n, by = C.c_double(), C.c_int64(), C.c_double()
            L.check(self._lib.acp_profile_read(self._ctx, k, C.byref(ms), C.byref(n), C.byref(by)))
            out[name] = {"ms": ms.value, "launches": n.value, "bytes": by.value}
        return out

    def check_finite(self, stream=None) -> None:
        """Synchronise and raise AcpError(ACP_E_NONFINITE) if a non-finite
        factor reached the orthogonaliser since creation."""
        L.check(self._lib.acp_check_finite(self._ctx, C.c_void_p(_stream_handle(stream))))

    def set_graphs(self, enable: bool = True) -> None:
        L.check(self._lib.acp_set_graphs(self._ctx, 1 if enable else 0))

    def launch_count(self) -> int:
        n = C.c_int64()
        L.check(self._lib.acp_launch_count(self._ctx, C.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.acp_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def verify_plan_across_ranks(plan: dict, group=None) -> bool:
    """True iff every rank of ``group`` derived the same fused-buffer plan
    (``plan_host`` / ``AcpContext.plan()``): ranks must issue identical bucket
    sequences, otherwise their all-reduces pair buckets of different
    sizes. Collective over any torch.distributed backend."""
    import hashlib
    import torch.distributed as dist
    digest = hashlib.sha256(repr((plan["tensors"], plan["buckets"])).encode()).hexdigest()
    got = [None] * dist.get_world_size(group)
    dist.all_gather_object(got, digest, group=group)
    return all(g == got[0] for g in got)
