"""compute-sanitizer memcheck / racecheck / synccheck over a tiny run of every
native kernel (SURVEY §4 "Sanitizers")."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.fail("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "17",
                        "--kernel-name", "kns=pspmm",  # our kernels (namespace pspmm), not torch's
                        sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses every run (exit 86):
        # runs under it have left GPUs needing a reset; nothing ran
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert "sanitize run ok" in out
    # memcheck / synccheck: "ERROR SUMMARY: 0 errors"; racecheck:
    # "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert ("ERROR SUMMARY: 0 errors" in out or
            "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out), out[-4000:]
