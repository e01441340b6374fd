import json, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2605_15695_b200 import api
import gen
g = bench.load_graph("reddit")
rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
cfg, A, _ = api.auto_select(rp, ci, vl, g.K)
B = torch.from_numpy(gen.config_B("reddit", g.n)).cuda(); C = torch.empty((g.n, g.K), device="cuda")
s = torch.cuda.Stream()
fb = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")
def flush():
    with torch.cuda.stream(s): fb.fill_(1.0)
with torch.cuda.stream(s):
    for steps in (20, 50, 200):
        for tag, fl in (("cold", flush), ("warm", lambda: None)):
            cs = bench.ClockSampler(0)
            ts = bench.time_steps(lambda: A.run(B, C, cfg, s), steps, 3, fl, s, cs)
            print(json.dumps({"steps": steps, "tag": tag, "median": float(np.median(ts)), "mean": float(np.mean(ts)),
                              "first5": [round(x, 4) for x in ts[:5]], "last5": [round(x, 4) for x in ts[-5:]], "clocks": cs.summary()}), flush=True)
