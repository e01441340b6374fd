"""NVLS multicast probe and single-rank check of pspmm_spmm_run_multicast
(f2 i over NVLS): a world-size-1 NCCL group, a symmetric-memory buffer
(torch.distributed._symmetric_memory) and its multicast address; the engine
writes C through multimem stores only, and the buffer (the rank's bound
copy) must then hold A.B.  Prints one JSON line; exit 0 with
"multicast": false when the box has no multicast support (the caller skips).

python tools/mc_probe.py [--port 29533]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    ap = argparse.ArgumentParser()
    ap.add_argument("--port", type=int, default=29533)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    out = {"device": torch.cuda.get_device_name(0)}
    try:
        import ctypes
        cu = ctypes.CDLL("libcuda.so.1")
        v = ctypes.c_int()
        # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
        cu.cuInit(0)
        cu.cuDeviceGetAttribute(ctypes.byref(v), 132, 0)
        out["driver_multicast_supported"] = int(v.value)
    except Exception as e:  # noqa: BLE001
        out["driver_multicast_supported"] = f"n/a: {e}"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(a.port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import gen
    import oracle
    from paper_2605_15695_b200 import api
    try:
        K = 64
        g = gen.config_graph("reddit", 0.004)
        buf = symm_mem.empty((g.n, K), dtype=torch.float32, device="cuda")
        hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
        mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
        out["torch_multicast_support"] = bool(hdl.has_multicast_support) if hasattr(
            hdl, "has_multicast_support") else None
        out["multicast_ptr"] = hex(mc)
        if not mc:
            out["multicast"] = False
            print(json.dumps(out))
            return 0
        out["multicast"] = True
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        B = gen.dense(g.n, K, 7)
        Bd = torch.from_numpy(B).cuda()
        ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=8)
        res = {}
        for name, (V, S, mode) in {"m0_v1s0": (1, 0, 0), "m0_v2s1": (2, 1, 0),
                                   "m0_v1s1": (1, 1, 0), "m3": (1, 0, 3)}.items():
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S)
            cfg = api.Config(W=4, F=2 if mode == 3 else 1, V=V, S=S, mode=mode,
                             G=8 if mode == 3 else 0)
            if mode == 0:
                cfg = api.Config(**{**api.auto_config(g.n, g.nnz, rp, ci, K).as_dict(),
                                    "V": V, "S": S, "mode": 0})
            buf.fill_(float("nan"))
            torch.cuda.synchronize()
            api.pspmm_spmm_run_multicast(A, Bd, buf, mc, cfg)
            torch.cuda.synchronize()
            got = buf.cpu().numpy().astype(np.float64)
            ok = np.abs(got - ref) <= 1e-5 * mag + 1e-6
            res[name] = bool(ok.all())
        for name, attach, mode, KK in (("m5", "blocks", 5, 128), ("m6", "band", 6, 64)):
            b2 = symm_mem.empty((g.n, KK), dtype=torch.float32, device="cuda")
            h2 = symm_mem.rendezvous(b2, dist.group.WORLD.group_name)
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
            if attach == "blocks":
                api.pspmm_pcsr_attach_blocks(A)
            else:
                api.pspmm_pcsr_attach_band(A, KK)
            B2 = gen.dense(g.n, KK, 9)
            b2.fill_(float("nan"))
            api.pspmm_spmm_run_multicast(A, torch.from_numpy(B2).cuda(), b2, int(h2.multicast_ptr),
                                         api.Config(mode=mode))
            torch.cuda.synchronize()
            r2, m2 = oracle.spmm(g.rowptr, g.colidx, g.val, B2, threads=8)
            got = b2.cpu().numpy().astype(np.float64)
            res[name] = bool((np.abs(got - r2) <= 1e-5 * m2 + 1e-6).all())
        out["parity"] = res
    finally:
        dist.destroy_process_group()
    print(json.dumps(out))
    return 0 if all(out.get("parity", {}).values()) else 1


if __name__ == "__main__":
    sys.exit(main())
