#!/usr/bin/env python
"""bench.py — ParamSpMM hot path on B200 (BASELINE.json metric: SpMM GFLOP/s
= 2 nnz K / t, achieved HBM GB/s, roofline fraction, speedup vs cuSPARSE, at
1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload reddit] [--headline-only]

One step = one pass of the whole hot path over the workload: at N = 1 the
engine call pspmm_spmm_run (zero_split + spmm kernels); at N > 1 each rank's
all-gather of B (NCCL) + its shard's pspmm_spmm_run (strong scaling: the
graph is fixed, its rows are split over the ranks).  PCSR build, features
and the decider are per-graph preprocessing (amortised) and are
outside the timed region.  Rank 0 prints ONE JSON line.

--impl reference times the repo's CPU oracle (oracle/, fp64 triple loop) on
a bounded row sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

PEAK_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)
L2_FLUSH_BYTES = 256 << 20


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(n_rows, n_cols, nnz, K):
    """R = A read once (int32 rowPtr + int32 colIdx + fp32 val) + B read once
    + C written once: 4(n+1) + 8 nnz + 4 n_cols K + 4 n_rows K."""
    return 4 * (n_rows + 1) + 8 * nnz + 4 * n_cols * K + 4 * n_rows * K


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: NVML every 2 ms in a thread (a ~30 ms timed region gets ~15
    samples), else `nvidia-smi -lms 100`."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, {reason names})
        self.stop = None
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device's own GPU, whatever the enumeration order
            import torch
            uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx),
                                             {k for k, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    self.stop.wait(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.stop = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.stop is not None:
            self.stop.set()
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        samples = list(self.samples)
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm, mx = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            samples.append((sm, mx, {nm for nm, v in zip(self.NAMES, parts[2:6])
                                     if v.lower().startswith("active")}))
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(r for _, _, r in samples))
        return {"sm_mhz": float(np.median([x[0] for x in samples])),
                "sm_max_mhz": float(max(x[1] for x in samples)),
                "reasons": sorted(reasons), "samples": len(samples),
                "source": "nvml 2 ms" if self.samples else "nvidia-smi 100 ms"}


# ----------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------
WORKLOADS = ["cora", "roadnet", "products", "proteins", "reddit", "proteins_clustered"]


def load_graph(name):
    cache = os.environ.get("PSPMM_GEN_CACHE")
    if cache:
        path = os.path.join(cache, f"{name}.npz")
        if os.path.exists(path):
            z = np.load(path)
            c = gen.CONFIGS[name]
            return gen.Graph(name, int(z["n"]), z["rowptr"], z["colidx"], z["val"], c["K"])
    g = gen.config_graph(name)
    if cache:
        os.makedirs(cache, exist_ok=True)
        np.savez(os.path.join(cache, f"{name}.npz"), n=g.n, rowptr=g.rowptr, colidx=g.colidx,
                 val=g.val)
    return g


def workload_desc(g):
    return f"{g.name}-shaped synthetic graph (n={g.n}, nnz={g.nnz}, K={g.K})"


def gather_roofline(name, head, K, ms):
    """The binding on-chip limit of the high-degree configs: B-row bytes
    gathered per launch (nnz_V vectors x K x 4; each vector fetches its B row
    once) against the measured bare-gather ceiling of the same pattern on
    this B200 (profiles/gather_ceiling.json, tools/microbench_gather.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_ceiling.json")) as f:
            ceil = json.load(f).get(name)
        nnz_v = head["pcsr"]["nnz_v"]
    except Exception:
        return None
    if not ceil:
        return None
    gathered = nnz_v * K * 4
    tbps = gathered / (ms * 1e-3) / 1e12
    return {"gathered_bytes_per_launch": gathered, "achieved_tbps": tbps,
            "ceiling_tbps": ceil["tbps"], "frac": tbps / ceil["tbps"], "source": ceil["source"]}


def traffic_for(name, cfg, cfg_dict=None):
    """ncu DRAM bytes per launch of the decided config (profiles/traffic.json),
    or None when the committed capture is of another config."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t.get(name)
        cd = cfg_dict if cfg_dict is not None else cfg.as_dict()
        if e and all(e["cfg"].get(k) == v for k, v in cd.items() if k in e["cfg"]):
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


# ----------------------------------------------------------------------------
# timing helpers
# ----------------------------------------------------------------------------
def time_steps(step, steps, warmup, flush, stream, sampler=None):
    """Per-step CUDA-event times (ms) on `stream`, L2 flushed between steps."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        for i in range(steps):
            flush()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def cusparse_best(g, rp, ci, vl, Bd, K, steps, flush, stream):
    """cusparseSpMM on the same device data: every CSR algorithm, best median."""
    import ctypes
    import torch
    from paper_2605_15695_b200 import build_ext
    try:
        lib = ctypes.CDLL(build_ext.LIB_CUSPARSE)
    except OSError as e:
        return {"error": str(e)}
    P = ctypes.c_void_p
    lib.pspmm_cusparse_create.argtypes = [ctypes.c_int64] * 3 + [P] * 4 + [
        ctypes.c_int64, ctypes.c_int32, P, ctypes.c_int64, ctypes.c_int32, P, ctypes.POINTER(P)]
    lib.pspmm_cusparse_run.argtypes = [P, P]
    lib.pspmm_cusparse_destroy.argtypes = [P]
    C = torch.empty((g.n, K), device="cuda")
    s = ctypes.c_void_p(stream.cuda_stream)
    res = {}
    names = {0: "ALG_DEFAULT", 1: "CSR_ALG1", 2: "CSR_ALG2", 3: "CSR_ALG3"}
    for alg in (0, 1, 2, 3):
        plan = P()
        st = lib.pspmm_cusparse_create(g.n, g.n, g.nnz, rp.data_ptr(), ci.data_ptr(),
                                       vl.data_ptr(), Bd.data_ptr(), K, K, C.data_ptr(), K, alg,
                                       s, ctypes.byref(plan))
        if st != 0:
            res[names[alg]] = {"status": st}
            continue
        try:
            # a comparison, not the headline: at most 20 steps per algorithm so a
            # large --steps keeps the run bounded (CSR_ALG1 takes ~0.1 s per
            # product on the big graphs)
            ts = time_steps(lambda: lib.pspmm_cusparse_run(plan, s), min(steps, 20), 3, flush,
                            stream)
            res[names[alg]] = {"ms": float(np.median(ts)), "min_ms": float(min(ts))}
        finally:
            torch.cuda.synchronize()
            lib.pspmm_cusparse_destroy(plan)
    del C
    ok = {k: v for k, v in res.items() if "ms" in v}
    best = min(ok, key=lambda k: ok[k]["ms"]) if ok else None
    return {"algs": res, "best": best, "best_ms": ok[best]["ms"] if best else None,
            "default_ms": ok.get("ALG_DEFAULT", {}).get("ms")}


def cpu_oracle_sample(g, B, target_s=12.0, threads=None):
    """Time the oracle (fp64 triple loop, OpenMP over rows) on a prefix of
    rows sized to ~target_s seconds; returns GFLOP/s over that sample."""
    import oracle
    threads = threads or os.cpu_count() or 1
    deg = np.cumsum(np.diff(g.rowptr.astype(np.int64)))
    K = B.shape[1]

    def run(rows):
        t0 = time.perf_counter()
        oracle.spmm(g.rowptr, g.colidx, g.val, B, rows=np.arange(rows, dtype=np.int64),
                    threads=threads, with_mag=False)
        return time.perf_counter() - t0

    # pilot on ~0.5% of the nonzeros, then scale to the target duration
    pilot_rows = int(np.searchsorted(deg, max(1, g.nnz // 200))) + 1
    pilot_rows = min(pilot_rows, g.n)
    tp = max(run(pilot_rows), 1e-4)
    nnz_p = int(deg[pilot_rows - 1])
    rate = nnz_p / tp
    want_nnz = int(min(g.nnz, rate * target_s))
    rows = min(g.n, int(np.searchsorted(deg, want_nnz)) + 1)
    t = run(rows)
    nnz_s = int(deg[rows - 1])
    return {"value": 2.0 * nnz_s * K / t / 1e9, "unit": "GFLOP/s", "cores": int(threads),
            "kind": "oracle",
            "sample": f"rows [0, {rows}) of {g.n} ({nnz_s} of {g.nnz} nnz, K={K}), "
                      f"{t:.1f} s wall, fp64 C = A.B only (oracle.spmm with_mag=False: the "
                      f"tolerance bound sum |a||b| is not computed)",
            "seconds": t}


# ----------------------------------------------------------------------------
# single-GPU workload measurement
# ----------------------------------------------------------------------------
def measure_single(g, steps, warmup, flush, stream, want_cusparse=True, want_e2e=True,
                   sampler=None):
    import torch
    from paper_2605_15695_b200 import api
    K = g.K
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    t0 = time.perf_counter()
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci, stream=stream)
    cfg = api.pspmm_decide_config(feats, K)
    t1 = time.perf_counter()
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override,
                             stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    A_dec, cfg0 = A, cfg
    # engine mode 1 (dense 128 x 32 tiles on tcgen05 + the rest): split once
    # per graph, taken when the tiles hold enough of A
    cfg, dense = api.auto_dense(A, rp, ci, vl, K, cfg, stream)
    if dense is not None:
        dense["dense_frac"] = dense["nnz_dense"] / max(1, g.nnz)
    # engine mode 5 (row blocks, B windows staged in shared memory): taken
    # when each staged B row would serve enough nonzeros (device-measured)
    cfg, A, blocks = api.auto_blocks(A, rp, ci, vl, K, cfg, stream)
    # engine mode 6 (staged bands): locality-ordered graphs whose 128-row
    # blocks' B-row ranges fit the shared-memory budget
    cfg, A, band = api.auto_band(A, rp, ci, vl, K, cfg, feats, stream)
    t3 = time.perf_counter()
    B = gen.config_B(g.name, g.n)
    Bd = torch.from_numpy(B).cuda()
    C = torch.empty((g.n, K), device="cuda")
    launches_per_step = 1 + (1 if (A.info["S"] == 1 and A.info["num_chunks"] > A.info["num_panels"]
                                   and cfg.mode != 5)
                             else 0) + (2 if cfg.mode == 1 else 0)  # mode 1: + split_b, dense_tc

    def step():
        A.run(Bd, C, cfg, stream)

    ts = time_steps(step, steps, warmup, flush, stream, sampler)
    ms = float(np.mean(ts))
    # SURVEY §8(d)'s primary leg: warm back-to-back launches (no flush; the
    # steady state of an iterative GNN), median, beside the cold mean above
    tw = time_steps(step, max(steps, 20), 2, lambda: None, stream)
    mode0 = None
    if cfg.mode in (1, 5, 6):  # the decider's own pick alone, for comparison
        c0 = api.Config(**(cfg.as_dict() if cfg.mode == 1 else cfg0.as_dict()))
        if cfg.mode == 1:
            c0.mode = 0
        A0 = A if cfg.mode == 1 else A_dec
        t0s = time_steps(lambda: A0.run(Bd, C, c0, stream), steps, warmup, flush, stream)
        mode0 = {"cfg": c0.as_dict(), "ms_median": float(np.median(t0s)),
                 "ms_mean": float(np.mean(t0s))}
    R = algorithmic_bytes(g.n, g.n, g.nnz, K)
    flops = 2.0 * g.nnz * K
    out = {
        "workload": workload_desc(g), "n": g.n, "nnz": g.nnz, "K": K,
        "cfg": cfg.as_dict(), "features": feats, "pcsr": {k: A.info[k] for k in
                                                           ("nnz_v", "num_chunks", "sg", "pr", "sr")},
        "ms_mean": ms, "ms_median": float(np.median(ts)), "ms_min": float(min(ts)),
        "warm_ms_median": float(np.median(tw)), "warm_ms_min": float(min(tw)),
        "gflops": flops / (ms * 1e-3) / 1e9, "algorithmic_bytes": R,
        "achieved_gbs": R / (ms * 1e-3) / 1e9, "launches_per_step": launches_per_step,
        "preprocess_s": {"features_decide": t1 - t0, "pcsr_build": t2 - t1,
                         "dense_split": t3 - t2},
    }
    if dense is not None:
        out["dense_split"] = dense
    if blocks is not None:
        out["row_blocks"] = blocks
    if band is not None:
        out["staged_band"] = band
    if mode0 is not None:
        out["mode0_same_knobs"] = mode0
    if want_cusparse:
        cs = cusparse_best(g, rp, ci, vl, Bd, K, steps, flush, stream)
        out["cusparse"] = cs
        if cs.get("best_ms"):
            out["speedup_vs_cusparse_best"] = cs["best_ms"] / out["ms_median"]
        if cs.get("default_ms"):
            out["speedup_vs_cusparse_default"] = cs["default_ms"] / out["ms_median"]
    if want_e2e:
        # a stream of products through the public host entry: every step
        # copies its B in from pinned host memory and its C out; two device
        # buffer sets rotate so step i+1's H2D and step i-1's D2H overlap
        # the engine on step i (pspmm_spmm_run_host_batch)
        hB = torch.from_numpy(B).pin_memory()
        hCs = [torch.empty((g.n, K)).pin_memory() for _ in range(2)]
        dBs = [Bd, torch.empty_like(Bd)]
        dCs = [C, torch.empty_like(C)]
        nb = max(3, steps)  # the same K steps as the device-timed region
        api.pspmm_spmm_run_host_batch(A, [hB] * 2, hCs, cfg, dBs, dCs, stream)  # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush()
        e0.record(stream)
        api.pspmm_spmm_run_host_batch(A, [hB] * nb, [hCs[i % 2] for i in range(nb)], cfg, dBs,
                                      dCs, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        me = e0.elapsed_time(e1) / nb
        # the single-product host entry (no cross-step overlap), for reference
        te = time_steps(lambda: api.pspmm_spmm_run_host(A, hB, hCs[0], cfg, Bd, C, stream),
                        3, 1, flush, stream)
        out["e2e"] = {"value": flops / (me * 1e-3) / 1e9, "unit": "GFLOP/s",
                      "h2d_bytes_per_step": int(B.nbytes), "d2h_bytes_per_step": int(g.n * K * 4),
                      "ms_per_step": me, "steps": nb,
                      "path": "pspmm_spmm_run_host_batch: per step pinned h_B -> H2D, "
                              "zero_split+spmm, D2H -> h_C; 2 rotating device buffer sets, "
                              "copies of neighbouring steps overlap the engine",
                      "single_call_ms": float(np.mean(te))}
    if want_e2e:
        # f3: one GNN layer H' = A H W with a K x K weight (SpMM + the dense
        # product), and the dense product alone
        Wd = torch.from_numpy(gen.dense(K, K, 4242)).cuda()
        T = torch.empty((g.n, K), device="cuda")
        Y = torch.empty((g.n, K), device="cuda")
        tl = time_steps(lambda: api.pspmm_gnn_layer(A, Bd, Wd, T, Y, cfg, stream), 5, 2, flush,
                        stream)
        tg = time_steps(lambda: api.pspmm_dense_gemm(Bd, Wd, T, stream), 5, 2, flush, stream)
        # the same bytes moved by a plain device copy: the practical ceiling
        # of a ~100 MB transfer (launch, ramp and drain included)
        tc = time_steps(lambda: T.copy_(Bd), 5, 2, flush, stream)
        ml, mg, mc = float(np.mean(tl)), float(np.mean(tg)), float(np.mean(tc))
        lf = 2.0 * g.nnz * K + 2.0 * g.n * K * K
        out["gnn_layer"] = {"ms": ml, "gflops": lf / (ml * 1e-3) / 1e9, "dense_gemm_ms": mg,
                            "dense_gemm_gbs": 8.0 * g.n * K / (mg * 1e-3) / 1e9,
                            "device_copy_ms": mc, "dense_gemm_over_copy": mc / mg,
                            "what": f"pspmm_gnn_layer: Y = A (X W), W {K}x{K}; flops 2 nnz K + "
                                    "2 n K^2; dense_gemm_gbs = X read + T written"}
    del A, A_dec, rp, ci, vl, Bd, C
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="reddit", choices=WORKLOADS)
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the per-config table of the other four workloads")
    ap.add_argument("--no-cusparse", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N>1: all-gather then SpMM, instead of overlapping the all-gather "
                         "with the own-column block")
    ap.add_argument("--exchange", default="auto",
                    choices=["auto", "allgather", "halo", "fanout", "multicast"],
                    help="N>1: row exchange (auto: halo when every rank references < 50 %% "
                         "of the remote rows, else the all-gather fused into the SpMM "
                         "epilogue (fanout) when the peers map over CUDA IPC, else the "
                         "overlapped NCCL all-gather)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to rehearse the N>1 flow on one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        # never time fewer ranks than asked: re-launch under torchrun when the
        # GPUs are there, else fail loudly
        if "WORLD_SIZE" in os.environ or args.gpus < 1:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) are "
                     f"visible; refusing to time fewer ranks than asked")
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), os.path.abspath(__file__)]
                 + sys.argv[1:])

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # single-GPU rehearsal of the multi-rank flow (not a measurement)
            dist.init_process_group("gloo")
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)

    peak, peak_src = hbm_peak()
    g = load_graph(args.workload)
    K = g.K
    sampler = ClockSampler(local_rank)

    if world == 1:
        with torch.cuda.stream(stream):
            head = measure_single(g, args.steps, args.warmup, flush, stream,
                                  want_cusparse=not args.no_cusparse, sampler=sampler)
        ms = head["ms_mean"]
        value = head["gflops"]
        launches = head["launches_per_step"] * args.steps
        cfg_d = head["cfg"]
        roof_ms = ms
        R = head["algorithmic_bytes"]
        e2e = head["e2e"]
    else:
        head, ms, roof_ms, R, cfg_d, launches, e2e = run_sharded(
            g, args, world, rank, stream, flush, sampler)
        value = 2.0 * g.nnz * K / (ms * 1e-3) / 1e9

    achieved = R / (roof_ms * 1e-3) / 1e9
    from paper_2605_15695_b200 import api
    # ncu DRAM traffic exists only for the single-GPU launch (ncu never wraps a
    # multi-rank command); a shard's traffic is not the 1-GPU figure
    traffic = traffic_for(args.workload, api.Config(**cfg_d)) if world == 1 else None
    line = {
        "metric": "SpMM GFLOP/s (2*nnz*K/t)",
        "value": value,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded generator gen/, shapes of the paper's workloads; DESIGN.md §4)",
        "config": {
            "workload": workload_desc(g), "n": g.n, "nnz": g.nnz, "K": K,
            "pcsr_config": cfg_d,
            "parallelism": "single GPU" if world == 1 else
                           f"{world}-way nnz-balanced row shards + "
                           f"{EXCHANGE_DESC[head.get('exchange', 'allgather')]}",
            "l2": "flushed between timed steps (256 MiB write, untimed)",
            "step": "pspmm_spmm_run (zero_split + spmm kernels)" if world == 1 else
                    head.get("step_desc"),
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "pspmm_spmm_run (zero_split_kernel + spmm_kernel)",
                     "algorithmic_bytes_per_launch": R,
                     "bytes_formula": "4(n+1) + 8 nnz + 4 n K (B once) + 4 n K (C once)",
                     "gather": gather_roofline(args.workload, head, K, roof_ms)},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if world == 1 and isinstance(head, dict):
        for k in ("cusparse", "speedup_vs_cusparse_best", "speedup_vs_cusparse_default",
                  "pcsr", "features", "preprocess_s", "ms_median", "ms_min", "gnn_layer"):
            if k in head:
                line[k] = head[k]
    if rank == 0 and world == 1:
        B = gen.config_B(g.name, g.n)
        line["cpu_baseline"] = cpu_oracle_sample(g, B)
        line["cpu_baseline"].pop("seconds", None)
        if not args.headline_only:
            per = []
            del g
            for name in WORKLOADS:
                if name == args.workload:
                    continue
                gg = load_graph(name)
                with torch.cuda.stream(stream):
                    r = measure_single(gg, args.steps, args.warmup, flush, stream,
                                       want_cusparse=not args.no_cusparse, want_e2e=False)
                r["roofline_frac"] = r["achieved_gbs"] / peak
                r["name"] = name
                # realised Table-3 features of every workload stay in the line
                per.append(r)
                del gg
            line["per_config"] = per
    # last key of the line (the driver keeps the line's tail): one compact
    # row per workload — engine config, cold mean / warm median ms, R-roofline
    # fraction, DRAM traffic over R (ncu, profiles/traffic.json), cuSPARSE
    if rank == 0:
        rows = [dict(head, name=args.workload)] if world == 1 else []
        rows += [dict(r, name=r.get("name", "")) for r in line.get("per_config", [])]
        line["summary"] = [summary_row(r, peak) for r in rows]
        if world > 1:
            line["summary"] = {"exchange_legs": head.get("exchange_legs")}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def cfg_str(c):
    return (f"m{c['mode']} V{c['V']} S{c['S']} W{c['W']} F{c['F']} G{c['G']}"
            + (f" o{c['order']}" if c.get("order") else ""))


def summary_row(r, peak):
    """One compact record of a measured workload (bench line summary)."""
    R = r["algorithmic_bytes"]
    tr = traffic_for(r["name"], None, r["cfg"])
    out = {"w": r["name"], "K": r["K"], "cfg": cfg_str(r["cfg"]), "ms": round(r["ms_mean"], 4),
           "warm_ms": round(r.get("warm_ms_median", float("nan")), 4),
           "frac": round(R / (r["ms_mean"] * 1e-3) / 1e9 / peak, 4),
           "dram_over_R": round(tr / R, 2) if tr else None}
    if r.get("speedup_vs_cusparse_best"):
        out["vs_cusparse"] = round(r["speedup_vs_cusparse_best"], 2)
    return out


def max_over_ranks(vals):
    """Element-wise max over ranks (device tensor on NCCL, host on gloo)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def run_sharded(g, args, world, rank, stream, flush, sampler):
    """N > 1: this rank's row shard of the fixed graph (strong scaling).  Step =
    exchange of B rows + local SpMM.  Every applicable exchange is timed as its
    own leg (`exchange_legs` in the line), each with its per-rank max step and
    kernel time and the bytes it moves per rank:
      allgather  NCCL all-gather of B overlapped with the own-column block
                 (the north star's row e; headline for dense halos such as the
                 shuffled Reddit-shaped graph)
      fanout     (f2 i) no collective: the SpMM epilogue stores every output
                 row into every rank's next-layer B over CUDA-IPC peer memory,
                 then a one-element all-reduce barrier
      halo       (f2 ii) all_to_all of only the referenced rows (headline for
                 locality-ordered graphs, where < 50 % of the remote rows are
                 referenced)
    --exchange X makes X the headline leg (and times only X)."""
    import torch
    from paper_2605_15695_b200 import api, dist as pdist
    K = g.K
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci, stream=stream)
    cfg = api.pspmm_decide_config(feats, K)
    del rp, ci
    B = gen.config_B(g.name, g.n)
    bounds = api.pspmm_shard_plan(g.rowptr, world, 2)
    (frac,) = max_over_ranks([pdist.halo_fraction(g.rowptr, g.colidx, bounds, rank)])
    if args.exchange != "auto":
        legs = [args.exchange]
    elif frac < 0.5:
        legs = ["halo", "allgather"]
    else:
        legs = ["allgather", "fanout", "multicast"]

    def launches(h):  # engine kernel + the split-panel zeroing kernel when present
        return 1 + (1 if (h.info["S"] == 1 and h.info["num_chunks"] > h.info["num_panels"])
                    else 0)

    def setup(kind):
        """-> dict(step, kernel_only, e2e_body, lo, rows, n_cols, nnz_loc, launches,
        desc, moved) or a string saying why the leg is unavailable."""
        if kind in ("fanout", "multicast"):
            run, note = setup_fanout(g, cfg, B, world, rank, stream, kind == "multicast")
            if run is None:
                return note or f"{kind} unavailable"
            sh = run.shard
            split = run.A.info["S"] == 1 and run.A.info["num_chunks"] > run.A.info["num_panels"]
            C_k = torch.empty((sh.rows, K), device="cuda")
            dB = torch.zeros((sh.n_max, K), device="cuda")

            def e2e_body(hB, hC):
                dB[:sh.rows].copy_(hB, non_blocking=True)
                pdist.all_gather_rows(dB, run.X[0])
                run.step(stream, swap=False)
                hC.copy_(run.own(1), non_blocking=True)
            return dict(
                step=lambda: run.step(stream, swap=False),
                kernel_only=lambda: run.A.run(run.X[0], C_k, cfg, stream),
                e2e_body=e2e_body, lo=sh.lo, rows=sh.rows, n_cols=sh.n_cols,
                nnz_loc=int(sh.rowptr[-1]), launches=1 + (world if split else 0),
                moved=(world - 1) * sh.rows * K * 4, keep=run,
                desc=("pspmm_spmm_run_multicast: SpMM whose epilogue writes each output element "
                      "ONCE with multimem.st to an NVSwitch multicast object binding every "
                      "rank's next-layer B (torch symmetric memory), then a one-element NCCL "
                      "all-reduce as the layer barrier" if kind == "multicast" else
                      "pspmm_spmm_run_fanout: SpMM whose epilogue stores each output row into "
                      "every rank's next-layer B (CUDA-IPC peer memory over NVLink), then a "
                      "one-element NCCL all-reduce as the layer barrier; no separate collective"))
        if kind == "halo":
            plan = pdist.make_halo_plan(g.rowptr, g.colidx, g.val, world, rank)
            with torch.cuda.stream(stream):
                run = pdist.HaloSpmm(plan, K, cfg, stream=stream)
            lo, rows = int(plan.bounds[rank]), plan.rows
            run.B_local.copy_(torch.from_numpy(B[lo:lo + rows]))

            def e2e_body(hB, hC):
                run.B_local.copy_(hB, non_blocking=True)
                run.step(stream)
                hC.copy_(run.C, non_blocking=True)
            return dict(
                step=lambda: run.step(stream),
                kernel_only=lambda: run.A.run(run.B_ext, run.C, cfg, stream),
                e2e_body=e2e_body, lo=lo, rows=rows, n_cols=rows + plan.n_halo,
                nnz_loc=int(plan.rowptr[-1]),
                launches=launches(run.A) + (1 if len(plan.send_idx) else 0),
                moved=int(plan.n_halo) * K * 4, keep=run,
                desc="halo all_to_all_single of the referenced B rows (row-gather pack) + SpMM")
        sh = pdist.make_shard(g.rowptr, g.colidx, g.val, world, rank, align=2)
        with torch.cuda.stream(stream):
            run = pdist.ShardedSpmm(sh, K, cfg, stream=stream)
        B_loc = pdist.pad_rows(torch.from_numpy(B[sh.lo:sh.lo + sh.rows]).cuda(), sh.n_max)
        overlap = not args.no_overlap and run.A_own is not None and args.dist_backend == "nccl"
        dB = torch.zeros((sh.n_max, K), device="cuda")

        def e2e_body(hB, hC):
            dB[:sh.rows].copy_(hB, non_blocking=True)
            run.step_overlap(dB, stream) if overlap else run.step(dB, stream)
            hC.copy_(run.C[:sh.rows], non_blocking=True)
        return dict(
            step=(lambda: run.step_overlap(B_loc, stream)) if overlap else
                 (lambda: run.step(B_loc, stream)),
            kernel_only=lambda: run.A.run(run.B_full, run.C, cfg, stream),
            e2e_body=e2e_body, lo=sh.lo, rows=sh.rows, n_cols=sh.n_cols,
            nnz_loc=int(sh.rowptr[-1]),
            launches=(launches(run.A_own) + (1 if run.A_rem is not None else 0)) if overlap
            else launches(run.A),
            moved=(world - 1) * sh.n_max * K * 4, keep=run,
            desc=("async all_gather_into_tensor(B) || own-column block SpMM, then "
                  "remote-column block pspmm_spmm_accumulate" if overlap else
                  "all_gather_into_tensor(B) then pspmm_spmm_run on the local shard"))

    results, head_leg = {}, None
    for i, kind in enumerate(legs):
        leg = setup(kind)
        if isinstance(leg, str):
            results[kind] = {"unavailable": leg}
            continue
        torch.cuda.synchronize()
        torch.distributed.barrier()
        with torch.cuda.stream(stream):
            ts = time_steps(leg["step"], args.steps, args.warmup, flush, stream,
                            sampler if head_leg is None else None)
            tk = time_steps(leg["kernel_only"], args.steps, 2, flush, stream)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        ms, kms = max_over_ranks([float(np.mean(ts)), float(np.mean(tk))])
        R = algorithmic_bytes(leg["rows"], leg["n_cols"], leg["nnz_loc"], K)
        (Rmax, moved_max) = max_over_ranks([float(R), float(leg["moved"])])
        results[kind] = {"ms": ms, "kernel_ms_max": kms,
                         "gflops": 2.0 * g.nnz * K / (ms * 1e-3) / 1e9,
                         "exchange_bytes_per_rank_max": int(moved_max),
                         "shard_algorithmic_bytes_max": int(Rmax),
                         "kernel_roofline_gbs": Rmax / (kms * 1e-3) / 1e9,
                         "launches_per_step": leg["launches"], "desc": leg["desc"]}
        if head_leg is None:
            head_leg = (kind, leg, ms, kms, Rmax)
        else:
            del leg
    if head_leg is None:
        raise RuntimeError(f"no exchange leg available: {results}")
    kind, leg, ms, kms, R = head_leg
    lo, rows = leg["lo"], leg["rows"]
    # e2e of the headline leg: pinned host B rows of this rank -> device,
    # exchange, SpMM, D2H of its C rows
    hB = torch.from_numpy(B[lo:lo + rows].copy()).pin_memory()
    hC = torch.empty((rows, K)).pin_memory()
    with torch.cuda.stream(stream):
        te = time_steps(lambda: leg["e2e_body"](hB, hC), max(3, min(args.steps, 10)), 2, flush,
                        stream)
    (me,) = max_over_ranks([float(np.mean(te))])
    e2e = {"value": 2.0 * g.nnz * K / (me * 1e-3) / 1e9, "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(hB.numel() * 4), "d2h_bytes_per_step": int(hC.numel() * 4),
           "ms_per_step": me, "path": f"rank shard ({kind}): H2D B rows, exchange, spmm, D2H C rows"}
    head = {"shard_rows": rows, "shard_nnz": leg["nnz_loc"], "kernel_ms_max": kms,
            "exchange": kind, "halo_fraction_max": frac, "step_desc": leg["desc"],
            "exchange_legs": results}
    return head, ms, kms, R, cfg.as_dict(), leg["launches"] * args.steps, e2e


EXCHANGE_DESC = {
    "halo": "halo all_to_all of the referenced B rows (NCCL)",
    "allgather": "all-gather of B rows (NCCL)",
    "fanout": "all-gather fused into the SpMM epilogue (P2P stores to every rank's next-layer "
              "B over CUDA IPC / NVLink)",
    "multicast": "all-gather fused into the SpMM epilogue as NVLS multimem stores (one store "
                 "per element, replicated by the NVSwitch)",
}


def setup_fanout(g, cfg, B, world, rank, stream, multicast=False):
    """Map every peer's gathered buffers (CUDA IPC) and validate one fused
    step against the plain engine on the same gathered input on all ranks.
    Returns (FanoutSpmm or None, note); every rank reaches the same decision
    (failures are max-reduced), so no rank is left waiting in a collective."""
    import torch
    from paper_2605_15695_b200 import api, dist as pdist
    sh = pdist.make_shard(g.rowptr, g.colidx, g.val, world, rank, align=2)
    with torch.cuda.stream(stream):
        run = (pdist.MulticastSpmm if multicast else pdist.FanoutSpmm)(sh, g.K, cfg, stream=stream)
    torch.cuda.synchronize()
    err = ""
    try:
        run.connect()
    except Exception as e:  # e.g. no P2P path between the GPUs
        err = f"connect: {e!r}"[:200]
    (bad,) = max_over_ranks([1.0 if err else 0.0])
    if bad:
        run.close()
        return None, err or "a peer rank failed to map the buffers"
    try:
        B_loc = pdist.pad_rows(torch.from_numpy(B[sh.lo:sh.hi].copy()).cuda(), sh.n_max)
        pdist.all_gather_rows(B_loc, run.X[0])
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            run.X[1].zero_()
            torch.cuda.synchronize()
            import torch.distributed as tdist
            tdist.barrier()
            run.step(stream, swap=False)
            mine = torch.empty((sh.rows, g.K), device="cuda")
            api.pspmm_spmm_run(run.A, run.X[0], mine, cfg, stream)
        torch.cuda.synchronize()
        # every slot of X[1] must hold its owner's rows: compare with the
        # all-gather of the plain engine's outputs
        ref = pdist.all_gather_rows(pdist.pad_rows(mine, sh.n_max))
        torch.cuda.synchronize()
        if not torch.allclose(run.X[1], ref, rtol=1e-4, atol=1e-4):
            err = "validation: fused copies differ from the all-gathered outputs"
    except Exception as e:
        err = f"validation: {e!r}"[:200]
    (bad,) = max_over_ranks([1.0 if err else 0.0])
    if bad:
        run.close()
        return None, err or "validation failed on a peer rank"
    return run, None


def run_reference(args, world, rank):
    """--impl reference: the oracle on the host cores, rank 0 only."""
    if rank != 0:
        return
    g = load_graph(args.workload)
    B = gen.config_B(g.name, g.n)
    per_step = []
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(g, B, target_s=budget)
        if i >= args.warmup:
            per_step.append(r)
    v = float(np.mean([r["value"] for r in per_step]))
    ms = float(np.mean([r["seconds"] for r in per_step])) * 1e3
    last = per_step[-1]
    line = {
        "impl": "reference", "metric": "SpMM GFLOP/s (2*nnz*K/t)", "value": v,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (gen/)",
        "config": {"workload": workload_desc(g), "n": g.n, "nnz": g.nnz, "K": g.K,
                   "parallelism": "host cores (OpenMP over rows)"},
        "cpu_baseline": {"kind": "oracle", "cores": last["cores"], "sample": last["sample"],
                         "value": v, "unit": "GFLOP/s"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
