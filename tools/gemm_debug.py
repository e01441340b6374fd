"""Locate wrong elements of the tensor-core dense product (tile / row /
chunk pattern) over X-ring depths, both forms (W in shared memory / W in
tensor memory) and tile counts per CTA."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_15695_b200 import api
    torch.manual_seed(0)
    for Ki, Ko in ((64, 64), (256, 64), (128, 128)):
        for n in (128 * 148 + 5, 128 * 148 * 3 + 77, 232965):
            X = torch.rand((n, Ki), device="cuda") * 2 - 1
            W = torch.rand((Ki, Ko), device="cuda") * 2 - 1
            ref = (X.double() @ W.double())
            for raw in ("2", "3", "8"):
                os.environ["PSPMM_GEMM_XS"] = raw
                T = torch.full((n, Ko), float("nan"), device="cuda")
                api.pspmm_dense_gemm(X, W, T)
                torch.cuda.synchronize()
                err = (T.double() - ref).abs()
                bad = torch.nonzero(err > 1e-3)
                rows = torch.unique(bad[:, 0]) if len(bad) else bad
                tiles = torch.unique(rows // 128) if len(rows) else rows
                print(f"Ki={Ki} Ko={Ko} n={n} xs={raw}: bad elems {len(bad)} rows {len(rows)} "
                      f"tiles {len(tiles)} first tiles {tiles[:8].tolist()} "
                      f"rows%128 {sorted(set((rows % 128).tolist()))[:12]} "
                      f"nan {int(torch.isnan(T).sum())}", flush=True)


if __name__ == "__main__":
    main()
