"""Multi-GPU path: nnz-balanced contiguous row
shards of A, one process per GPU, and an all-gather of B before every SpMM —
the GNN-layer pattern where layer l's output rows become layer l+1's B rows.

Host logic (shard plan, column remap into the padded all-gather layout) is in
the C library (pspmm_shard_plan / pspmm_shard_extract); the collective is
torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU tests);
the compute is pspmm_spmm_run on the rank's PCSR.  This module never imports
the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import api


class _nvtx:
    """NVTX range around a multi-GPU step phase (exchange / SpMM), so an
    Nsight Systems timeline shows how the collective overlaps the engine
    (SURVEY §5); a no-op where NVTX is unavailable."""

    def __init__(self, name):
        self.name = name
        self.on = False

    def __enter__(self):
        try:
            import torch
            torch.cuda.nvtx.range_push(self.name)
            self.on = True
        except Exception:
            pass
        return self

    def __exit__(self, *exc):
        if self.on:
            import torch
            torch.cuda.nvtx.range_pop()
        return False


@dataclass
class Shard:
    rank: int
    world: int
    bounds: np.ndarray   # P + 1 row bounds (int64)
    n_max: int           # padded rows per rank in the gathered B
    rowptr: np.ndarray   # local CSR, rows bounds[r]..bounds[r+1]
    colidx: np.ndarray   # columns remapped to owner * n_max + offset
    val: np.ndarray

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def n_cols(self) -> int:
        return self.world * self.n_max


def make_shard(rowptr, colidx, val, world: int, rank: int, align: int = 2) -> Shard:
    """Row shard of rank `rank` (align = panel height so V = 2 panels never
    straddle two ranks)."""
    bounds = api.pspmm_shard_plan(rowptr, world, align)
    lrp, lci, lvl, n_max = api.pspmm_shard_extract(rowptr, colidx, val, world, bounds, rank)
    return Shard(rank, world, bounds, n_max, lrp, lci, lvl)


def pad_rows(x_local, n_max: int):
    """Pad this rank's B rows to n_max (all-gather needs equal counts)."""
    import torch
    if x_local.shape[0] == n_max:
        return x_local
    out = torch.zeros((n_max,) + tuple(x_local.shape[1:]), dtype=x_local.dtype,
                      device=x_local.device)
    out[: x_local.shape[0]] = x_local
    return out


def all_gather_rows(x_padded, out=None, group=None):
    """B_full[g * n_max + i] = rank g's row i.  NCCL: one
    all_gather_into_tensor; gloo (CPU tests): all_gather into a list."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world * x_padded.shape[0],) + tuple(x_padded.shape[1:]),
                          dtype=x_padded.dtype, device=x_padded.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, x_padded, group=group)
    elif x_padded.is_cuda:
        # gloo (CPU tests / single-GPU rehearsal of the multi-rank bench):
        # stage through host memory
        host = torch.empty((world * x_padded.shape[0],) + tuple(x_padded.shape[1:]),
                           dtype=x_padded.dtype)
        dist.all_gather(list(host.split(x_padded.shape[0])), x_padded.cpu(), group=group)
        out.copy_(host)
    else:
        parts = list(out.split(x_padded.shape[0]))
        dist.all_gather(parts, x_padded, group=group)
    return out


def local_rows(x_full, shard: Shard):
    """This rank's rows of a gathered matrix (inverse of the padding)."""
    start = shard.rank * shard.n_max
    return x_full[start:start + shard.rows]


def unpad_gathered(x_full, bounds, n_max: int):
    """Gathered (P n_max) x K -> the n x K matrix in original row order."""
    import torch
    parts = [x_full[g * n_max: g * n_max + int(bounds[g + 1] - bounds[g])]
             for g in range(len(bounds) - 1)]
    return torch.cat(parts, 0)


class ShardedSpmm:
    """One rank's state for C_r = A[r-rows, :] . B (B gathered every step)."""

    def __init__(self, shard: Shard, K: int, cfg: api.Config | None = None, device="cuda",
                 stream=None):
        import torch
        self.shard = shard
        self.K = K
        rp = torch.from_numpy(shard.rowptr).to(device)
        ci = torch.from_numpy(shard.colidx if len(shard.colidx) else np.zeros(1, np.int32)).to(device)
        vl = torch.from_numpy(shard.val if len(shard.val) else np.zeros(1, np.float32)).to(device)
        nnz = int(shard.rowptr[-1])
        if cfg is None:
            cfg = api.Config(W=4, F=1, V=1, S=1)
        self.cfg = cfg
        self.A = api.pspmm_pcsr_build(shard.rows, nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega,
                                      cfg.sg_override, stream, n_cols=shard.n_cols)
        # overlap split: the own-column block needs only this rank's B rows,
        # so it runs while the all-gather of the peers' rows is in flight
        own, rem = split_own_columns(shard)
        self.A_own = self.A_rem = None
        if own[2].shape[0] and shard.world > 1:
            self.A_own = _build(own, shard.rows, shard.rows, cfg, device, stream)
            if rem[2].shape[0]:
                self.A_rem = _build(rem, shard.rows, shard.n_cols, cfg, device, stream)
        self.B_full = torch.empty((shard.n_cols, K), dtype=torch.float32, device=device)
        self.C = torch.empty((shard.n_max, K), dtype=torch.float32, device=device)
        self.C[shard.rows:].zero_()

    def step(self, B_padded, stream=None, group=None):
        """All-gather the padded B shards, then the local SpMM.  Returns the
        padded local C (the next layer's B shard)."""
        with _nvtx("pspmm allgather"):
            all_gather_rows(B_padded, self.B_full, group)
        with _nvtx("pspmm spmm"):
            self.A.run(self.B_full, self.C, self.cfg, stream)
        return self.C

    def step_overlap(self, B_padded, stream=None, group=None):
        """Same result as step(): C = A_own . B_local while NCCL gathers the
        peers' rows, then C += A_rem . B_full (pspmm_spmm_accumulate)."""
        import torch.distributed as dist
        if self.A_own is None or dist.get_backend(group) != "nccl":
            return self.step(B_padded, stream, group)
        with _nvtx("pspmm allgather || own-column spmm"):
            work = dist.all_gather_into_tensor(self.B_full, B_padded, group=group,
                                               async_op=True)
            self.A_own.run(B_padded, self.C, self.cfg, stream)
            work.wait()  # the compute stream waits for the gathered rows
        if self.A_rem is not None:
            with _nvtx("pspmm remote-column spmm"):
                api.pspmm_spmm_accumulate(self.A_rem, self.B_full, self.C, self.cfg, stream)
        return self.C


class FanoutSpmm:
    """f2 (i): the all-gather fused into the SpMM epilogue.

    Each rank holds two gathered buffers X[0], X[1] (P n_max x K each, one
    allocation, double-buffered across layers).  A layer reads X[cur] and the
    engine (pspmm_spmm_run_fanout) writes its output rows into slot `rank` of
    X[1 - cur] on EVERY rank — its own copy plus P - 1 peer stores issued from
    the epilogue as rows complete (NVLink P2P through CUDA-IPC mappings) — so
    no collective follows the SpMM; a stream-ordered barrier (one-element
    NCCL all-reduce) makes the peers' rows visible before the next layer.

    connect(group) maps the peers' buffers (CUDA IPC, handles exchanged with
    all_gather_object); connect_local(others) wires simulated ranks that live
    in one process (single-GPU tests)."""

    def __init__(self, shard: Shard, K: int, cfg: api.Config | None = None, device="cuda",
                 stream=None):
        import torch
        self.shard = shard
        self.K = K
        self.cfg = cfg if cfg is not None else api.Config(W=4, F=1, V=1, S=1)
        rp, ci, vl = shard.rowptr, shard.colidx, shard.val
        self.A = _build((rp, ci if len(ci) else np.zeros(1, np.int32),
                         vl if len(vl) else np.zeros(1, np.float32)),
                        shard.rows, shard.n_cols, self.cfg, device, stream)
        self.XX = torch.zeros((2, shard.n_cols, K), dtype=torch.float32, device=device)
        self.X = [self.XX[0], self.XX[1]]
        self.cur = 0
        self.peers = [[], []]   # per buffer: device addresses of slot `rank` at each peer
        self._opened = []
        self._flag = None

    @property
    def slot_bytes(self) -> int:
        return self.shard.rank * self.shard.n_max * self.K * 4

    def own(self, b: int):
        """This rank's rows of buffer b (a view; also what peers receive)."""
        s = self.shard
        return self.X[b][s.rank * s.n_max: s.rank * s.n_max + s.rows]

    def connect(self, group=None):
        import torch.distributed as dist
        handle, off = api.pspmm_ipc_get_handle(self.XX)
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, (handle, off), group=group)
        buf_bytes = self.shard.n_cols * self.K * 4
        bases = {}
        for q, (h, o) in enumerate(allh):
            if q == self.shard.rank:
                continue
            if h not in bases:
                bases[h] = api.pspmm_ipc_open(h)
                self._opened.append(bases[h])
            for b in (0, 1):
                self.peers[b].append(bases[h] + o + b * buf_bytes + self.slot_bytes)

    def connect_local(self, others):
        """Simulated ranks in one process: others = the FanoutSpmm of every
        other rank (same device)."""
        for b in (0, 1):
            self.peers[b] = [o.X[b].data_ptr() + self.slot_bytes for o in others]

    def load(self, X_full):
        """Initial layer input (the gathered B, P n_max x K) into X[cur]."""
        self.X[self.cur].copy_(X_full)

    def barrier(self, group=None):
        import torch
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            if self._flag is None:
                self._flag = torch.zeros(1, dtype=torch.float32, device=self.XX.device)
            dist.all_reduce(self._flag, group=group)  # stream-ordered
        else:
            torch.cuda.synchronize()
            dist.barrier(group=group)

    def step(self, stream=None, group=None, swap=True, barrier=True):
        """One layer: own rows of X[1 - cur] (and their copies at every peer)
        = A_shard . X[cur].  swap=False keeps reading X[0] (fixed-input
        benchmarking).  Returns this rank's output rows."""
        src, dst = self.cur, 1 - self.cur
        out = self.own(dst)
        with _nvtx("pspmm spmm + fan-out stores"):
            api.pspmm_spmm_run_fanout(self.A, self.X[src], out, self.peers[dst], self.cfg,
                                      stream, K=self.K)
        if swap:
            self.cur = dst
        if barrier:
            with _nvtx("pspmm layer barrier"):
                self.barrier(group)
        return out

    def close(self):
        for b in self._opened:
            try:
                api.pspmm_ipc_close(b)
            except Exception:
                pass
        self._opened = []
        self.peers = [[], []]


class MulticastSpmm(FanoutSpmm):
    """f2 (i) over NVLS: the fan-out of FanoutSpmm with ONE multimem store per
    C write.  The two gathered buffers live in one symmetric-memory
    allocation (torch.distributed._symmetric_memory) whose NVSwitch
    multicast object binds every rank's copy; the engine
    (pspmm_spmm_run_multicast) writes each output element once to the
    multicast address of slot `rank` and the switch replicates it into every
    rank's buffer (the rank's own included).  connect() raises if the group
    has no multicast support (the caller falls back to FanoutSpmm)."""

    def __init__(self, shard: Shard, K: int, cfg: api.Config | None = None, device="cuda",
                 stream=None):
        super().__init__(shard, K, cfg, device, stream)
        self._mc = None

    def connect(self, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        g = group if group is not None else dist.group.WORLD
        XX = symm_mem.empty((2, self.shard.n_cols, self.K), dtype=self.XX.dtype,
                            device=self.XX.device)
        XX.zero_()
        hdl = symm_mem.rendezvous(XX, g.group_name)
        mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
        if not mc:
            raise RuntimeError("MulticastSpmm: no NVSwitch multicast for this group")
        self._hdl = hdl
        self.XX = XX
        self.X = [XX[0], XX[1]]
        buf_bytes = self.shard.n_cols * self.K * 4
        self._mc = [mc + b * buf_bytes + self.slot_bytes for b in (0, 1)]

    def connect_local(self, others):
        raise NotImplementedError("MulticastSpmm needs a multicast object (connect)")

    def step(self, stream=None, group=None, swap=True, barrier=True):
        src, dst = self.cur, 1 - self.cur
        out = self.own(dst)
        with _nvtx("pspmm spmm + multimem stores"):
            api.pspmm_spmm_run_multicast(self.A, self.X[src], out, self._mc[dst], self.cfg,
                                         stream)
        if swap:
            self.cur = dst
        if barrier:
            with _nvtx("pspmm layer barrier"):
                self.barrier(group)
        return out

    def close(self):
        self._mc = None


def split_own_columns(shard: Shard):
    """Local CSR split into (own, remote) column blocks, both canonical:
    own = columns owned by this rank, remapped to local row indices of B
    (col - rank * n_max); remote = the other columns, in the gathered layout.
    Each is (rowptr, colidx, val) numpy."""
    lo = shard.rank * shard.n_max
    ci = shard.colidx.astype(np.int64)
    mine = (ci >= lo) & (ci < lo + shard.rows)
    deg = np.diff(shard.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(shard.rows), deg)

    def part(mask, shift):
        counts = np.bincount(rows[mask], minlength=shard.rows)
        rp = np.zeros(shard.rows + 1, np.int64)
        np.cumsum(counts, out=rp[1:])
        return (rp.astype(np.int32), (ci[mask] - shift).astype(np.int32), shard.val[mask])

    return part(mine, lo), part(~mine, 0)


def _build(part, n_rows, n_cols, cfg, device, stream):
    import torch
    rp, ci, vl = part
    return api.pspmm_pcsr_build(
        n_rows, int(rp[-1]), torch.from_numpy(rp).to(device), torch.from_numpy(ci).to(device),
        torch.from_numpy(vl).to(device), cfg.V, cfg.S, cfg.omega, cfg.sg_override, stream,
        n_cols=n_cols)


# ---------------------------------------------------------------------------
# Halo exchange (SURVEY §8(f) f2 ii): each rank receives only the B rows its
# shard's columns reference, instead of the whole all-gathered B.  For a
# locality-ordered graph (roadNet: columns within ~sqrt(n) of the row) the
# halo is a thin band at each shard boundary; for a shuffled power-law graph
# it approaches all of B and the all-gather (NCCL's fastest collective) wins,
# so `halo_fraction` lets the caller choose.
# ---------------------------------------------------------------------------
@dataclass
class HaloPlan:
    rank: int
    world: int
    bounds: np.ndarray      # P + 1 row bounds
    rows: int               # local rows
    rowptr: np.ndarray      # local CSR with columns in [0, rows + n_halo)
    colidx: np.ndarray
    val: np.ndarray
    recv_counts: list       # rows received from each peer (halo, owner order)
    send_idx: np.ndarray    # local row ids to send, peers concatenated in rank order
    send_counts: list

    @property
    def n_halo(self) -> int:
        return int(sum(self.recv_counts))


def halo_fraction(rowptr, colidx, bounds, rank) -> float:
    """Halo rows / remote rows for this rank's shard (1.0 = needs all of B)."""
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    cols = np.asarray(colidx[rowptr[lo]:rowptr[hi]], dtype=np.int64)
    remote = cols[(cols < lo) | (cols >= hi)]
    n_remote = int(bounds[-1]) - (hi - lo)
    return len(np.unique(remote)) / max(1, n_remote)


def _halo_local(rowptr, colidx, val, bounds, rank):
    """This rank's side of the plan: local CSR over [own rows | halo] (canonical)
    and the halo rows it needs, as (owner, owner-local row) ascending."""
    world = len(bounds) - 1
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    base = int(rowptr[lo])
    lrp = (np.asarray(rowptr[lo:hi + 1], dtype=np.int64) - base)
    cols = np.asarray(colidx[base:int(rowptr[hi])], dtype=np.int64)
    vals = np.asarray(val[base:int(rowptr[hi])], dtype=np.float32)
    remote = (cols < lo) | (cols >= hi)
    need = np.unique(cols[remote])                       # ascending = owner order
    owner = np.searchsorted(bounds, need, side="right") - 1
    recv_counts = np.bincount(owner, minlength=world).astype(np.int64)
    # local column ids: own rows first, then the halo in `need` order
    new_cols = np.where(remote, (hi - lo) + np.searchsorted(need, cols), cols - lo)
    # keep the local CSR canonical: re-sort every row by its new column ids
    lrows = np.repeat(np.arange(hi - lo, dtype=np.int64), np.diff(lrp))
    order = np.argsort(lrows * (hi - lo + len(need) + 1) + new_cols, kind="stable")
    new_cols, vals = new_cols[order], vals[order]
    req_local = (need - bounds[owner]).astype(np.int64)
    return (hi - lo, lrp.astype(np.int32), new_cols.astype(np.int32), vals, recv_counts,
            req_local)


def make_halo_plan(rowptr, colidx, val, world: int, rank: int, group=None,
                   align: int = 2) -> HaloPlan:
    """Host preprocessing, once per graph: the rank's rows, the remote rows it
    needs (grouped by owner, ascending), and — via one all_to_all of counts
    and one of indices — the rows each peer needs from it."""
    import torch
    import torch.distributed as dist
    bounds = api.pspmm_shard_plan(rowptr, world, align)
    rows, lrp, cols, vals, recv_counts, req_local = _halo_local(rowptr, colidx, val, bounds, rank)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    cnt_out = torch.from_numpy(recv_counts.copy()).to(dev)
    cnt_in = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(cnt_in, cnt_out, group=group)
    send_counts = cnt_in.cpu().numpy().astype(np.int64)
    idx_in = torch.empty(int(send_counts.sum()), dtype=torch.int64, device=dev)
    dist.all_to_all_single(idx_in, torch.from_numpy(req_local).to(dev),
                           output_split_sizes=send_counts.tolist(),
                           input_split_sizes=recv_counts.tolist(), group=group)
    return HaloPlan(rank, world, bounds, rows, lrp, cols, vals, recv_counts.tolist(),
                    idx_in.cpu().numpy().astype(np.int32), send_counts.tolist())


def simulate_halo_plans(rowptr, colidx, val, world: int, align: int = 2):
    """All ranks' HaloPlans computed in one process (the request exchange done
    by transposing the lists) — single-GPU tests of the halo path."""
    bounds = api.pspmm_shard_plan(rowptr, world, align)
    local = [_halo_local(rowptr, colidx, val, bounds, r) for r in range(world)]
    plans = []
    for r in range(world):
        rows, lrp, cols, vals, recv_counts, _ = local[r]
        send_idx, send_counts = [], []
        for q in range(world):  # rows rank q asks from rank r, in q's order
            rq, req = local[q][4], local[q][5]
            start = int(rq[:r].sum())
            part = req[start:start + int(rq[r])]
            send_idx.append(part)
            send_counts.append(len(part))
        plans.append(HaloPlan(r, world, bounds, rows, lrp, cols, vals, recv_counts.tolist(),
                              np.concatenate(send_idx).astype(np.int32), send_counts))
    return plans


class HaloSpmm:
    """One rank's C_r = A[r-rows, :] . B with a halo exchange per step:
    pack the rows peers asked for (pspmm_permute_rows as a row gather),
    all_to_all_single them, SpMM over [local rows | halo rows]."""

    def __init__(self, plan: HaloPlan, K: int, cfg: api.Config | None = None, device="cuda",
                 stream=None):
        import torch
        self.plan = plan
        self.K = K
        cfg = cfg or api.Config(W=4, F=1, V=1, S=1)
        self.cfg = cfg
        nnz = int(plan.rowptr[-1])
        self.A = api.pspmm_pcsr_build(
            plan.rows, nnz, torch.from_numpy(plan.rowptr).to(device),
            torch.from_numpy(plan.colidx if nnz else np.zeros(1, np.int32)).to(device),
            torch.from_numpy(plan.val if nnz else np.zeros(1, np.float32)).to(device),
            cfg.V, cfg.S, cfg.omega, cfg.sg_override, stream, n_cols=plan.rows + plan.n_halo)
        # B_ext = [local rows | halo]; the next layer writes its C into the first part
        self.B_ext = torch.zeros((plan.rows + plan.n_halo, K), dtype=torch.float32, device=device)
        self.send_idx = torch.from_numpy(plan.send_idx.astype(np.int32)).to(device)
        self.send_buf = torch.empty((max(1, len(plan.send_idx)), K), dtype=torch.float32,
                                    device=device)
        self.C = torch.empty((plan.rows, K), dtype=torch.float32, device=device)

    @property
    def B_local(self):
        return self.B_ext[: self.plan.rows]

    def exchange(self, group=None, stream=None):
        import torch
        import torch.distributed as dist
        p = self.plan
        if len(p.send_idx):
            api.pspmm_permute_rows(self.B_local, self.send_idx, inverse=True,
                                   out=self.send_buf[: len(p.send_idx)], stream=stream)
        halo = self.B_ext[p.rows:]
        if dist.get_backend(group) == "nccl":
            dist.all_to_all_single(halo, self.send_buf[: len(p.send_idx)],
                                   output_split_sizes=p.recv_counts,
                                   input_split_sizes=p.send_counts, group=group)
        else:  # gloo: host staging
            out = torch.empty((p.n_halo, self.K), dtype=torch.float32)
            dist.all_to_all_single(out, self.send_buf[: len(p.send_idx)].cpu(),
                                   output_split_sizes=p.recv_counts,
                                   input_split_sizes=p.send_counts, group=group)
            halo.copy_(out)

    def step(self, stream=None, group=None):
        """B_local must hold this layer's input rows; returns C (rows x K)."""
        with _nvtx("pspmm halo exchange"):
            self.exchange(group, stream)
        with _nvtx("pspmm spmm"):
            self.A.run(self.B_ext, self.C, self.cfg, stream)
        return self.C
