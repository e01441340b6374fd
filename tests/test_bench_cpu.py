"""bench.py host-side contract checks that need no GPU."""
import os
import subprocess
import sys

from conftest import ROOT


def test_bench_gpus_without_torchrun_fails_loudly():
    """`python bench.py --gpus 2` must never time fewer ranks than asked: on a
    box without enough GPUs it exits non-zero and prints no JSON line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "cora"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "refusing to time fewer ranks" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
