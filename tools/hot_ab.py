"""A/B: split the B gather's L2 policy by row hotness.

After a descending-degree reordering (P A P^T, f1) the most-gathered B rows
are the lowest row ids; rows < H are loaded with L2 evict_last, the rest
with evict_first (experimental knob pspmm_x_set_hot_cols).  Prints one JSON
line per (workload, ordering, config, H) with the median / min ms.

python tools/hot_ab.py --workloads products,reddit
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import gen
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="products,reddit")
    ap.add_argument("--iters", type=int, default=9)
    ap.add_argument("--fracs", default="-1,0,0.25,0.5,0.75,1.0,1.5")
    a = ap.parse_args()
    lib = api._lib
    lib.pspmm_x_set_hot_cols.argtypes = [ctypes.c_int64]
    lib.pspmm_x_set_hot_cols.restype = None
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for w in a.workloads.split(","):
        g = bench.load_graph(w)
        rp0 = torch.from_numpy(g.rowptr).cuda()
        ci0 = torch.from_numpy(g.colidx).cuda()
        vl0 = torch.from_numpy(g.val).cuda()
        B0 = torch.from_numpy(gen.config_B(g.name, g.n)).cuda()
        K = g.K
        for ordering in ("as_generated", "degree"):
            if ordering == "degree":
                perm = api.pspmm_reorder(g.rowptr, g.colidx, "degree")
                pd = torch.from_numpy(perm).cuda()
                rp, ci, vl = api.pspmm_csr_permute(rp0, ci0, vl0, pd)
                B = api.pspmm_permute_rows(B0, pd)
            else:
                rp, ci, vl, B = rp0, ci0, vl0, B0
            torch.cuda.synchronize()
            C = torch.empty((g.n, K), device="cuda")
            for (F, G) in ((2, 16), (1, 32), (1, 16)):
                if 4 * F * G > K and (F, G) != (1, K // 4):
                    continue
                cfg = api.Config(W=2, F=F, V=1, S=0, G=G, order=1)
                A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
                for fr in [float(x) for x in a.fracs.split(",")]:
                    H = -1 if fr < 0 else int(fr * l2 / (4 * K))
                    lib.pspmm_x_set_hot_cols(H)
                    ts = bench.time_steps(lambda: A.run(B, C, cfg), a.iters, 3, flush, stream)
                    print(json.dumps({"workload": w, "ordering": ordering, "F": F, "G": G,
                                      "hot_frac_of_l2": fr, "hot_rows": H,
                                      "ms": float(np.median(ts)), "min_ms": float(min(ts))}),
                          flush=True)
                lib.pspmm_x_set_hot_cols(-1)
                A.close()
            del C


if __name__ == "__main__":
    main()
