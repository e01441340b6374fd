"""NVLS multicast probe and single-rank check of pspmm_spmm_run_multicast
(f2 i over NVLS).  The multicast object comes from torch symmetric memory
when the group gives one (torch skips multicast for a one-rank group), else
straight from the driver's multicast API (cuMulticastCreate with this one
device bound, cuMemCreate + cuMulticastBindMem, unicast and multicast
mappings).  The engine writes C through multimem stores only, and the bound
physical memory (read through the unicast mapping) must then hold A.B.
Prints one JSON line; exit 0 with "multicast": false when the box has no
multicast support (the caller skips).

python tools/mc_probe.py [--port 29533]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class DriverMulticast:
    """One multicast object with device 0 bound (CUDA driver API via ctypes):
    .uc = unicast address of the bound memory, .mc = its multicast address."""

    def __init__(self, nbytes):
        import ctypes as C
        cu = C.CDLL("libcuda.so.1")
        self.cu = cu

        def ck(r, what):
            if r != 0:
                raise RuntimeError(f"{what} -> CUresult {r}")

        class Loc(C.Structure):
            _fields_ = [("type", C.c_int), ("id", C.c_int)]

        class McProp(C.Structure):
            _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t),
                        ("handleTypes", C.c_ulonglong), ("flags", C.c_ulonglong)]

        class AllocFlags(C.Structure):
            _fields_ = [("compressionType", C.c_ubyte), ("gpuDirectRDMACapable", C.c_ubyte),
                        ("usage", C.c_ushort), ("reserved", C.c_ubyte * 4)]

        class AllocProp(C.Structure):
            _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc),
                        ("win32HandleMetaData", C.c_void_p), ("allocFlags", AllocFlags)]

        class AccessDesc(C.Structure):
            _fields_ = [("location", Loc), ("flags", C.c_int)]

        ck(cu.cuInit(0), "cuInit")
        dev = C.c_int()
        ck(cu.cuDeviceGet(C.byref(dev), 0), "cuDeviceGet")
        # handle types: POSIX fd (1), none (0), fabric (8); the first the driver takes
        self.mch = C.c_ulonglong()
        tried = []
        for ht in (1, 0, 8):
            mp = McProp(1, nbytes, ht, 0)
            gran = C.c_size_t()
            r = cu.cuMulticastGetGranularity(C.byref(gran), C.byref(mp), 1)
            if r != 0:
                tried.append((ht, "granularity", r))
                continue
            size = (nbytes + gran.value - 1) // gran.value * gran.value
            mp.size = size
            r = cu.cuMulticastCreate(C.byref(self.mch), C.byref(mp))
            tried.append((ht, "create", r))
            if r == 0:
                break
        else:
            raise RuntimeError(f"cuMulticastCreate failed: {tried}")
        self.tried = tried
        ck(cu.cuMulticastAddDevice(self.mch, dev), "cuMulticastAddDevice")
        ap = AllocProp(1, 0, Loc(1, 0), None, AllocFlags())
        mg = C.c_size_t()
        ck(cu.cuMemGetAllocationGranularity(C.byref(mg), C.byref(ap), 0), "mem granularity")
        size = (size + mg.value - 1) // mg.value * mg.value
        self.mem = C.c_ulonglong()
        ck(cu.cuMemCreate(C.byref(self.mem), C.c_size_t(size), C.byref(ap), C.c_ulonglong(0)),
           "cuMemCreate")
        ck(cu.cuMulticastBindMem(self.mch, C.c_size_t(0), self.mem, C.c_size_t(0),
                                 C.c_size_t(size), C.c_ulonglong(0)), "cuMulticastBindMem")
        acc = AccessDesc(Loc(1, 0), 3)
        ptrs = []
        for handle in (self.mem, self.mch):
            p = C.c_ulonglong()
            ck(cu.cuMemAddressReserve(C.byref(p), C.c_size_t(size), C.c_size_t(gran.value),
                                      C.c_ulonglong(0), C.c_ulonglong(0)), "reserve")
            ck(cu.cuMemMap(p, C.c_size_t(size), C.c_size_t(0), handle, C.c_ulonglong(0)), "map")
            ck(cu.cuMemSetAccess(p, C.c_size_t(size), C.byref(acc), C.c_size_t(1)), "access")
            ptrs.append(p.value)
        self.uc, self.mc, self.size = ptrs[0], ptrs[1], size


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
        buf = symm_mem.empty((g.n, 128), dtype=torch.float32, device="cuda")
        hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
        mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
        out["torch_multicast_support"] = bool(hdl.has_multicast_support) if hasattr(
            hdl, "has_multicast_support") else None
        out["multicast_ptr"] = hex(mc)
        if not mc:
            try:
                drv = DriverMulticast(g.n * 128 * 4)
                out["source"] = "driver (cuMulticastCreate, 1 device bound)"
            except Exception as e:  # noqa: BLE001
                out["multicast"] = False
                out["driver_error"] = str(e)[:200]
                print(json.dumps(out))
                return 0
        else:
            drv = None
            out["source"] = "torch symmetric memory"
        out["multicast"] = True
        import ctypes as C
        cu = C.CDLL("libcuda.so.1")
        if drv is not None:
            uc, mcp = drv.uc, drv.mc
        else:
            big = symm_mem.empty((g.n, 128), dtype=torch.float32, device="cuda")
            hb = symm_mem.rendezvous(big, dist.group.WORLD.group_name)
            uc, mcp = big.data_ptr(), int(hb.multicast_ptr)
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        stream = torch.cuda.current_stream()

        def run_mc(A, Bn, cfg):
            """C (n x K at the bound memory, ld = K) via multimem only."""
            KK = Bn.shape[1]
            Bd = torch.from_numpy(Bn).cuda()
            torch.cuda.synchronize()
            assert cu.cuMemsetD32_v2(C.c_ulonglong(uc), C.c_uint(0x7FC00000),
                                     C.c_size_t(g.n * KK)) == 0
            st = api._lib.pspmm_spmm_run_multicast(A.handle, C.c_void_p(Bd.data_ptr()), KK, KK,
                                                   C.c_void_p(uc), KK, C.c_void_p(mcp), cfg,
                                                   C.c_void_p(stream.cuda_stream))
            assert st == 0, api._lib.pspmm_last_error()
            torch.cuda.synchronize()
            h = np.empty((g.n, KK), np.float32)
            assert cu.cuMemcpyDtoH_v2(h.ctypes.data_as(C.c_void_p), C.c_ulonglong(uc),
                                      C.c_size_t(h.nbytes)) == 0
            return h.astype(np.float64)

        res = {}
        B = gen.dense(g.n, K, 7)
        ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=8)
        for name, (V, S, mode) in {"m0_v1s0": (1, 0, 0), "m0_v2s1": (2, 1, 0),
                                   "m0_v1s1": (1, 1, 0), "m3": (1, 0, 3)}.items():
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S)
            cfg = api.Config(W=4, F=2, V=V, S=S, mode=3, G=8)
            if mode == 0:
                cfg = api.Config(**{**api.auto_config(g.n, g.nnz, rp, ci, K).as_dict(),
                                    "V": V, "S": S, "mode": 0})
            got = run_mc(A, B, cfg)
            res[name] = bool((np.abs(got - ref) <= 1e-5 * mag + 1e-6).all())
        for name, attach, mode, KK in (("m5", "blocks", 5, 128), ("m6", "band", 6, 64)):
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
            if attach == "blocks":
                api.pspmm_pcsr_attach_blocks(A)
            else:
                api.pspmm_pcsr_attach_band(A, KK)
            B2 = gen.dense(g.n, KK, 9)
            got = run_mc(A, B2, api.Config(mode=mode))
            r2, m2 = oracle.spmm(g.rowptr, g.colidx, g.val, B2, threads=8)
            res[name] = bool((np.abs(got - r2) <= 1e-5 * m2 + 1e-6).all())
        out["parity"] = res
    finally:
        dist.destroy_process_group()
    print(json.dumps(out))
    return 0 if all(out.get("parity", {}).values()) else 1


if __name__ == "__main__":
    sys.exit(main())
