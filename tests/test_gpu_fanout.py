"""(f2 i) The all-gather fused into the SpMM epilogue (pspmm_spmm_run_fanout,
dist.FanoutSpmm): every rank's output rows land in every rank's gathered
buffer.  Single-GPU coverage: (1) simulated ranks in one process whose
"peers" are each other's buffers on the same device — every copy must match
the full-graph oracle (c-5) for all engines and PCSR corners; (2) two real
processes on the same GPU mapping each other's buffers with CUDA IPC — the
same code path as NVLink peers, minus the link."""
import os
import socket

import numpy as np
import pytest

import gen
from gpu_util import assert_parity, oracle_ref

pytestmark = pytest.mark.gpu

K = 64


def _cases():
    out = []
    for mode in (0, 2, 3):
        for V, S in ((1, 0), (1, 1), (2, 0), (2, 1)):
            if mode == 3 and (V, S) != (1, 0):
                continue
            out.append((mode, V, S))
    return out


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("mode,V,S", _cases())
def test_fanout_simulated_ranks(P, mode, V, S):
    import torch
    from paper_2605_15695_b200 import api, dist
    g = gen.config_graph("reddit", 0.01)
    B = gen.dense(g.n, K, 5005)
    ref, mag = oracle_ref(g, B, key=("reddit_s_dist", K))
    shards = [dist.make_shard(g.rowptr, g.colidx, g.val, P, r, align=2) for r in range(P)]
    n_max = shards[0].n_max
    Bd = torch.from_numpy(B).cuda()
    B_full = torch.cat([dist.pad_rows(Bd[s.lo:s.hi], n_max) for s in shards], 0)
    cfg = api.Config(V=V, S=S, W=4, mode=mode, F=1)
    runs = [dist.FanoutSpmm(s, K, cfg) for s in shards]
    for r, run in enumerate(runs):
        run.connect_local([o for q, o in enumerate(runs) if q != r])
        run.X[1].fill_(float("nan"))      # every row must be (re)written
        run.load(B_full)
    # padded rows are never written: zero them as the real buffers start
    for run in runs:
        for q, s in enumerate(shards):
            run.X[1][q * n_max + s.rows:(q + 1) * n_max].zero_()
    for run in runs:
        run.step(barrier=False)
    torch.cuda.synchronize()
    for r, run in enumerate(runs):
        assert run.cur == 1
        C_full = dist.unpad_gathered(run.X[1], shards[0].bounds, n_max)
        assert_parity(C_full.cpu().numpy(), ref, mag, f"fanout P{P} m{mode} V{V} S{S} copy {r}")
        for q, s in enumerate(shards):
            assert not run.X[1][q * n_max + s.rows:(q + 1) * n_max].any()
    # layer 2 (double buffer): the fan-out chain's second product against the
    # fp64 oracle of A times the exact layer-1 output the GPU produced (its
    # fp32 rows are layer 2's input), element by element with the c-1 bound
    X1 = dist.unpad_gathered(runs[0].X[1], shards[0].bounds, n_max).cpu().numpy()
    for run in runs:
        run.step(barrier=False)
    torch.cuda.synchronize()
    ref2, mag2 = oracle_ref(g, np.ascontiguousarray(X1, np.float32))
    for r, run in enumerate(runs):
        assert run.cur == 0
        C2 = dist.unpad_gathered(run.X[0], shards[0].bounds, n_max)
        assert_parity(C2.cpu().numpy(), ref2, mag2, f"fanout layer 2 P{P} m{mode} V{V} S{S} "
                                                     f"copy {r}")


def test_fanout_argument_errors():
    import torch
    from paper_2605_15695_b200 import api
    g = gen.uniform(1000, 8, 3)
    from gpu_util import dev
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    B = torch.rand((g.n, 16), device="cuda")
    C = torch.empty((g.n, 16), device="cuda")
    peers = [torch.empty((g.n, 16), device="cuda") for _ in range(8)]
    with pytest.raises(ValueError):
        api.pspmm_spmm_run_fanout(A, B, C, peers, api.Config(V=1, S=0))
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_spmm_run_fanout(A, B, C, [0], api.Config(V=1, S=0))
    assert e.value.status == 1  # PSPMM_ERR_INVALID_ARG (null peer)
    with pytest.raises(api.PspmmError):  # peer alignment differs from C's
        api.pspmm_spmm_run_fanout(A, B, C, [peers[0].data_ptr() + 4], api.Config(V=1, S=0))
    # zero peers == pspmm_spmm_run
    api.pspmm_spmm_run_fanout(A, B, C, [], api.Config(V=1, S=0))
    C2 = torch.empty_like(C)
    api.pspmm_spmm_run(A, B, C2, api.Config(V=1, S=0))
    torch.cuda.synchronize()
    assert torch.equal(C, C2)
    # seven peers (the maximum): every copy bit-identical to C (S = 0: plain stores)
    api.pspmm_spmm_run_fanout(A, B, C, peers[:7], api.Config(V=1, S=0))
    torch.cuda.synchronize()
    for p in peers[:7]:
        assert torch.equal(p, C)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, S, q):
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import gen as g_
        from paper_2605_15695_b200 import api, dist
        g = g_.config_graph("reddit", 0.005)
        B = g_.dense(g.n, K, 4242)
        sh = dist.make_shard(g.rowptr, g.colidx, g.val, world, rank, align=2)
        run = dist.FanoutSpmm(sh, K, api.Config(V=1, S=S, W=4))
        run.connect()
        Bd = torch.from_numpy(B[sh.lo:sh.hi].copy()).cuda()
        run.load(dist.all_gather_rows(dist.pad_rows(Bd, sh.n_max)))
        tdist.barrier()
        run.step()               # gloo barrier: synchronize + barrier
        X = run.X[1].cpu().numpy()
        run.close()
        q.put((rank, "ok", X, sh.bounds, sh.n_max))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "err", repr(e), None, None))
        raise
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("S", [0, 1])
def test_fanout_ipc_two_processes(S):
    """Two processes on one GPU, buffers mapped with pspmm_ipc_open: each
    rank's gathered output holds both ranks' rows (c-5)."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, S, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] == "ok", r[2]
    g = gen.config_graph("reddit", 0.005)
    B = gen.dense(g.n, K, 4242)
    ref, mag = oracle_ref(g, B)
    import torch
    from paper_2605_15695_b200 import dist
    for rank, _, X, bounds, n_max in res:
        C = dist.unpad_gathered(torch.from_numpy(X), bounds, n_max).numpy()
        assert_parity(C, ref, mag, f"ipc rank {rank} S{S}")
