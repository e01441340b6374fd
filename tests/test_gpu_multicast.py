"""(f2 i over NVLS) pspmm_spmm_run_multicast: every C write is one multimem
store / reduction to a multicast address (torch symmetric memory on a
world-size-1 NCCL group); the rank's bound copy must equal the fp64 oracle
for engine modes 0 (V x S corners, split-panel multimem reductions), 3, 5
and 6.  Skipped when the box exposes no NVSwitch multicast object."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_multicast_epilogue_single_rank():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "mc_probe.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(lines[-1])
    if not out.get("multicast"):
        pytest.skip(f"no NVSwitch multicast on this box: {out}")
    assert r.returncode == 0 and all(out["parity"].values()), out
