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
