"""bench.py end to end on the GPU (small workload): the single-GPU JSON line
carries the contract keys, and the N>1 flow (row shards + all-gather + max
over ranks) runs as a 2-rank rehearsal on one GPU with the gloo backend
(NCCL cannot put two ranks on one device)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
        "clocks")


def _run(cmd, env=None):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    out = _run([sys.executable, "bench.py", "--workload", "cora", "--steps", "3", "--warmup", "3",
                "--headline-only"])
    for k in KEYS:
        assert k in out, k
    assert out["n_gpus"] == 1 and out["value"] > 0 and out["gpu_launches"] >= 3
    assert set(out["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert set(out["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert out["cpu_baseline"]["kind"] == "oracle" and out["cpu_baseline"]["cores"] >= 1
    assert "with_mag=False" in out["cpu_baseline"]["sample"]
    # the compact per-workload summary is the line's LAST key (the driver keeps the tail)
    assert list(out)[-1] == "summary" and out["summary"][0]["w"] == "cora"
    assert out["summary"][0]["warm_ms"] > 0


def test_bench_refuses_more_gpus_than_visible():
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--workload", "cora"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k != "WORLD_SIZE"})
    assert r.returncode != 0 and "refusing" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.parametrize("exchange,port", [("allgather", 29533), ("halo", 29534)])
def test_bench_two_rank_rehearsal_gloo(exchange, port):
    out = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py",
                "--workload", "cora", "--steps", "3", "--warmup", "3", "--headline-only",
                "--dist-backend", "gloo", "--exchange", exchange])
    assert out["n_gpus"] == 2 and out["value"] > 0
    assert "row shards" in out["config"]["parallelism"]
    assert ("halo" in out["config"]["parallelism"]) == (exchange == "halo")
    assert list(out["summary"]["exchange_legs"]) == [exchange]
    assert out["roofline"]["traffic"] is None  # no 1-GPU ncu figure on a shard


def test_bench_two_rank_auto_times_both_legs():
    """--exchange auto on a dense-halo graph: the all-gather (row e, headline)
    and the epilogue fan-out (f2 i) are both timed and reported; the NVLS
    multicast leg is listed (unavailable under gloo / without a multicast
    object, with its reason)."""
    out = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                "--master-addr", "127.0.0.1", "--master-port", "29535", "bench.py",
                "--workload", "cora", "--steps", "3", "--warmup", "3", "--headline-only",
                "--dist-backend", "gloo"])
    legs = out["summary"]["exchange_legs"]
    assert list(legs) == ["allgather", "fanout", "multicast"]
    assert "ms" in legs["multicast"] or "unavailable" in legs["multicast"], legs
    for k in ("allgather", "fanout"):
        assert legs[k]["ms"] > 0 and legs[k]["kernel_ms_max"] > 0, legs
        assert legs[k]["exchange_bytes_per_rank_max"] > 0


def test_bench_reference_arm():
    out = _run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cora",
                "--steps", "2", "--warmup", "1"])
    assert out["impl"] == "reference" and out["value"] > 0
    assert out["e2e"]["h2d_bytes_per_step"] == 0
