"""CPU-side checks of the boundary: the shared library loads without a GPU and
exports every entry point include/acp.h declares; the binding's struct
layout matches the header; host-side validation rejects bad configs."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT, ensure_built

HEADER = os.path.join(ROOT, "include", "acp.h")


def _lib_path():
    return os.path.join(ROOT, "paper_2306_08881_b200", "lib", "libacp.so")


@pytest.fixture(scope="module")
def lib():
    ensure_built()  # nvcc cross-compiles; no GPU needed
    from paper_2306_08881_b200 import _lib
    return _lib.load()


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(acp_[a-z0-9_]+)\s*\(", txt)))


def test_header_declarations_exported(lib):
    names = _declared()
    assert "acp_create" in names and "acp_step" in names and "acp_destroy" in names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in acp.h but not exported"
    from paper_2306_08881_b200._lib import EXPORTED
    assert sorted(EXPORTED) == names


def test_symbols_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib_path()], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for n in _declared():
        assert n in syms, n


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_struct_layout(lib):
    from paper_2306_08881_b200._lib import AcpConfig
    # offsets implied by acp.h on LP64
    assert AcpConfig.rows.offset == 8
    assert AcpConfig.nccl_comm.offset == 32
    assert AcpConfig.q0_host.offset == 48
    assert AcpConfig.workspace.offset == 72
    assert C.sizeof(AcpConfig) == 88


def test_abi_version_and_invalid_config(lib):
    from paper_2306_08881_b200._lib import AcpConfig, ACP_E_INVAL
    assert lib.acp_abi_version() == 1
    out = C.c_size_t()
    assert lib.acp_workspace_bytes(None, C.byref(out)) == ACP_E_INVAL
    cfg = AcpConfig()
    cfg.abi_version = 99
    assert lib.acp_workspace_bytes(C.byref(cfg), C.byref(out)) == ACP_E_INVAL
    assert b"abi" in lib.acp_last_error()
    assert lib.acp_step(None, 0, None, None) == ACP_E_INVAL


def test_plan_only_context_matches_oracle_plan(lib):
    """acp_plan_create builds the plan with no GPU; its offsets and buckets
    equal the oracle's independent restatement (C7-C10) bit for
    bit, and every call that needs device state is refused (ACP_E_STATE)."""
    from paper_2306_08881_b200 import plan_host
    from paper_2306_08881_b200._lib import AcpConfig, ACP_E_STATE, ACP_ABI_VERSION
    from oracle import fusion_plan
    from acp_inputs import ready_order
    for model, rank, bb in [("resnet50", 4, 25 * 2 ** 20), ("bert-base", 8, 25 * 2 ** 20),
                            ("resnet152", 4, 0), ("resnet152", 4, -1), ("resnet152", 4, 2 ** 20)]:
        shapes = [s for _, s in ready_order(model)]
        got = plan_host(shapes, rank, bucket_bytes=bb)
        want = fusion_plan(shapes, rank, bb)
        for i, (r, po, qo, eo, bp, bq) in enumerate(got["tensors"]):
            L = want["layers"][i]
            assert (r, po, qo, eo) == (L.r, want["slot_off"][0][i], want["slot_off"][1][i], want["e_off"][i])
            assert i in want["buckets"][0][bp] and i in want["buckets"][1][bq]
        for parity in (0, 1):
            assert len(got["buckets"][parity]) == len(want["buckets"][parity])
            for (off, cnt), members in zip(got["buckets"][parity], want["buckets"][parity]):
                first, last = members[0], members[-1]
                assert off == want["slot_off"][parity][first]
                end = (want["slot_off"][parity][last + 1] if last + 1 < len(shapes)
                       else want["arena_elems"][parity])
                assert off + cnt == end
    # device calls on a plan-only context
    rows = (C.c_int64 * 2)(64, 10)
    cols = (C.c_int64 * 2)(32, 0)
    cfg = AcpConfig()
    cfg.abi_version = ACP_ABI_VERSION
    cfg.num_tensors = 2
    cfg.rows = C.cast(rows, C.POINTER(C.c_int64))
    cfg.cols = C.cast(cols, C.POINTER(C.c_int64))
    cfg.rank = 4
    cfg.world_size = 2
    cfg.device = -1
    ctx = C.c_void_p()
    assert lib.acp_plan_create(C.byref(cfg), C.byref(ctx)) == 0
    assert lib.acp_step(ctx, 0, None, None) == ACP_E_STATE
    assert b"plan-only" in lib.acp_last_error()
    assert lib.acp_check_finite(ctx, None) == ACP_E_STATE
    assert lib.acp_get_state(ctx, 0, None, None, None, None) == ACP_E_STATE
    assert lib.acp_step_begin(ctx, 0, None, None) == ACP_E_STATE
    assert lib.acp_destroy(ctx) == 0
