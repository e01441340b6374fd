"""World-size-2 gloo test of the multi-GPU host path (shard plan, column
remap into the padded all-gather layout, the all-gather itself and the
un-padding).  The per-rank SpMM is the oracle here (CPU), so this checks the
plumbing; the GPU parity of the same path is tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import oracle
        from paper_2605_15695_b200 import dist as pdist
        g = gen.config_graph("reddit", 0.004)
        K = 8
        B = gen.dense(g.n, K, 77)
        sh = pdist.make_shard(g.rowptr, g.colidx, g.val, world, rank, align=2)
        # layer 1: gather B, local SpMM (oracle on the remapped shard)
        B_local = torch.from_numpy(B[sh.lo:sh.hi].copy())
        B_full = pdist.all_gather_rows(pdist.pad_rows(B_local, sh.n_max))
        C_local, _ = oracle.spmm(sh.rowptr, sh.colidx, sh.val, B_full.numpy())
        # layer 2: the output rows are the next layer's B shard
        B2_full = pdist.all_gather_rows(pdist.pad_rows(torch.from_numpy(
            C_local.astype(np.float32)), sh.n_max))
        C2_local, _ = oracle.spmm(sh.rowptr, sh.colidx, sh.val, B2_full.numpy())
        C2 = pdist.all_gather_rows(pdist.pad_rows(torch.from_numpy(C2_local), sh.n_max))
        full = pdist.unpad_gathered(C2, sh.bounds, sh.n_max).numpy()
        if rank == 0:
            ref1, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B)
            ref2, _ = oracle.spmm(g.rowptr, g.colidx, g.val, ref1.astype(np.float32))
            q.put(("ok", float(np.abs(full - ref2).max()), sh.bounds.tolist(), g.n))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_layer_chain():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    status, err, bounds, n = q.get(timeout=5)
    assert status == "ok", err
    assert err == 0.0  # same per-row fp64 sums, just relocated
    assert bounds[0] == 0 and bounds[-1] == n and bounds[1] % 2 == 0
    assert all(p.exitcode == 0 for p in procs)


def _halo_worker(rank, world, port, q, name):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import oracle
        from paper_2605_15695_b200 import dist as pdist
        g = gen.config_graph(name, 0.004 if name == "reddit" else 0.002)
        K = 8
        B = gen.dense(g.n, K, 99)
        plan = pdist.make_halo_plan(g.rowptr, g.colidx, g.val, world, rank)
        lo = int(plan.bounds[rank])
        B_local = B[lo:lo + plan.rows]
        # the exchange HaloSpmm performs, with a numpy row gather as the pack
        send = torch.from_numpy(np.ascontiguousarray(B_local[plan.send_idx]))
        halo = torch.empty((plan.n_halo, K))
        dist.all_to_all_single(halo, send, output_split_sizes=plan.recv_counts,
                               input_split_sizes=plan.send_counts)
        B_ext = np.concatenate([B_local, halo.numpy()], 0)
        C_local, _ = oracle.spmm(plan.rowptr, plan.colidx, plan.val, B_ext)
        ref, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B,
                             rows=np.arange(lo, lo + plan.rows, dtype=np.int64))
        frac = pdist.halo_fraction(g.rowptr, g.colidx, plan.bounds, rank)
        for i in range(plan.rows):  # the local CSR stays canonical
            assert np.all(np.diff(plan.colidx[plan.rowptr[i]:plan.rowptr[i + 1]]) > 0)
        q.put(("ok", rank, float(np.abs(C_local - ref).max()), plan.n_halo, frac))
    except Exception as e:  # pragma: no cover
        q.put(("err", rank, repr(e), 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["roadnet", "reddit"])
def test_two_rank_gloo_halo_exchange(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 2, port, q, name)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = [q.get(timeout=5) for _ in range(2)]
    for status, rank, err, n_halo, frac in res:
        assert status == "ok", err
        assert err < 1e-12  # same fp64 products, summed in the re-sorted column order
    if name == "roadnet":  # locality order: a thin halo at the shard boundary
        assert all(r[4] < 0.05 for r in res)
    assert all(p.exitcode == 0 for p in procs)


def _fanout_worker(rank, world, port, q):
    """FanoutSpmm.connect's host logic with the CUDA IPC calls stubbed: the
    handle exchange, one mapping per distinct peer allocation, and the peer
    slot addresses (base + tensor offset + buffer b + this rank's slot)."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        from paper_2605_15695_b200 import api
        from paper_2605_15695_b200 import dist as pdist
        g = gen.config_graph("reddit", 0.002)
        K = 8
        sh = pdist.make_shard(g.rowptr, g.colidx, g.val, world, rank, align=2)
        run = object.__new__(pdist.FanoutSpmm)
        run.shard, run.K = sh, K
        run.XX = torch.zeros((2, sh.n_cols, K))
        run.peers, run._opened = [[], []], []
        opened = []
        api.pspmm_ipc_get_handle = lambda t: (bytes([65 + rank]) * 64, 4096 * (rank + 1))
        api.pspmm_ipc_open = lambda h: opened.append(h) or (h[0] - 64) << 40
        run.connect()
        buf = sh.n_cols * K * 4
        want = [[((q + 1) << 40) + 4096 * (q + 1) + b * buf + rank * sh.n_max * K * 4
                 for q in range(world) if q != rank] for b in (0, 1)]
        q.put(("ok", rank, run.peers == want, len(opened) == world - 1))
    except Exception as e:  # pragma: no cover
        q.put(("err", rank, repr(e), False))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_fanout_peer_addresses(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fanout_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = [q.get(timeout=5) for _ in range(world)]
    for status, rank, ok_addr, ok_open in res:
        assert status == "ok", ok_addr
        assert ok_addr is True and ok_open is True
    assert all(p.exitcode == 0 for p in procs)
