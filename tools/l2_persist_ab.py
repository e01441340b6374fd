"""A/B: pin B in L2 with a stream access-policy window (persisting lines)
versus the engine's per-load evict_last policy alone.  Reddit-shaped
workload, decided config; one JSON line per variant (median / min ms).

python tools/l2_persist_ab.py --workload reddit
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from cuda.bindings import runtime as rt

    import bench
    import gen
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="reddit")
    ap.add_argument("--iters", type=int, default=15)
    a = ap.parse_args()
    g = bench.load_graph(a.workload)
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    cfg = api.auto_config(g.n, g.nnz, rp, ci, g.K)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
    B = torch.from_numpy(gen.config_B(a.workload, g.n)).cuda()
    C = torch.empty((g.n, g.K), device="cuda")
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")

    def flush():
        # persisting lines survive a plain flush: demote them first, so each
        # timed step starts with B out of L2 like the other variant
        rt.cudaCtxResetPersistingL2Cache()
        flush_buf.fill_(1.0)

    prop = torch.cuda.get_device_properties(0)
    err, max_persist = rt.cudaDeviceGetAttribute(
        rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
    err, max_window = rt.cudaDeviceGetAttribute(
        rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
    print(json.dumps({"l2": prop.L2_cache_size, "max_persisting": max_persist,
                      "max_window": max_window, "B_bytes": B.numel() * 4, "cfg": cfg.as_dict()}),
          flush=True)
    s = stream.cuda_stream

    def run(tag):
        with torch.cuda.stream(stream):
            ts = bench.time_steps(lambda: A.run(B, C, cfg, stream), a.iters, 5, flush, stream)
        print(json.dumps({"variant": tag, "ms": float(np.median(ts)), "min_ms": float(min(ts))}),
              flush=True)

    run("evict_last only")
    for frac in (0.5, 1.0):
        size = min(int(B.numel() * 4), max_window)
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize,
                              min(max_persist, int(size * frac) + (1 << 20)))
        attr = rt.cudaStreamAttrValue()
        attr.accessPolicyWindow.base_ptr = B.data_ptr()
        attr.accessPolicyWindow.num_bytes = size
        attr.accessPolicyWindow.hitRatio = frac
        attr.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
        attr.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
        r = rt.cudaStreamSetAttribute(s, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow,
                                      attr)
        print(json.dumps({"set_window": str(r[0]), "hit_ratio": frac, "bytes": size}), flush=True)
        run(f"persisting window hitRatio {frac}")
        attr.accessPolicyWindow.num_bytes = 0
        rt.cudaStreamSetAttribute(s, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow,
                                  attr)
        rt.cudaCtxResetPersistingL2Cache()


if __name__ == "__main__":
    main()
