"""compute-sanitizer over every kernel class at tiny shapes (SURVEY §5,
VERDICT r01 weak #9): memcheck (out-of-bounds / misaligned global and shared
accesses), racecheck (shared-memory hazards inside a CTA: the TMA ring, the
row-group reductions, K2's staging) and synccheck (illegal barrier use).
A round-1 cross-SM stale-L1 race in K2 was found only by a full-size parity
test; these tools check the intra-CTA half of that class directly."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tests", "sanitize_run.py")]
    if tool == "memcheck":
        cmd[1:1] = ["--leak-check", "no"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-6000:]
    assert "sanitize ok" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
