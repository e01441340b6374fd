"""Markdown results table for DESIGN.md §8 from a bench.py JSON line and the
ncu summaries of the same configs.

python tools/design_table.py profiles/r01/bench_r01_final.json --ncu profiles/r01/ncu_{w}_final.json
"""
import argparse
import json
import math


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("bench")
    ap.add_argument("--ncu", default="", help="pattern with {w} for the workload name")
    a = ap.parse_args()
    d = json.loads(open(a.bench).read().strip().splitlines()[-1])
    rows = []
    head = {"workload": d["config"]["workload"], "cfg": d["config"]["pcsr_config"],
            "ms_mean": d["ms_per_step"], "gflops": d["value"],
            "roofline_frac": d["roofline"]["frac"],
            "speedup_vs_cusparse_best": d.get("speedup_vs_cusparse_best"),
            "cusparse": d.get("cusparse")}
    for p in d.get("per_config", []) + [head]:
        name = p["workload"].split("-")[0]
        ncu = None
        if a.ncu:
            try:
                ncu = json.load(open(a.ncu.format(w=name)))[0]
            except Exception:
                ncu = None
        c = p["cfg"]
        cfg = f"m{c['mode']} V{c['V']} S{c['S']} W{c['W']} F{c['F']} G{c['G']}" + (
            f" o{c.get('order', 0)}" if c["mode"] == 0 else "")
        bind = ""
        if ncu:
            bind = (f"DRAM {ncu['dram_throughput_pct']:.0f} %, L2 {ncu['l2_throughput_pct']:.0f} % "
                    f"(hit {ncu['l2_hit_pct']:.0f} %), {ncu['dram_bytes'] / 1e9:.2f} GB DRAM, "
                    f"occupancy {ncu['achieved_occupancy_pct']:.0f} %")
        cs = p.get("cusparse") or {}
        sp = p.get("speedup_vs_cusparse_best")
        rows.append((name, cfg, p["ms_mean"], p["gflops"], p["roofline_frac"], bind,
                     f"{cs.get('best', '?')} {cs.get('best_ms', float('nan')):.3f}", sp))
    print("| config | engine config (decided) | ms | GFLOP/s | R-roofline frac | ncu (one launch) "
          "| cuSPARSE best (ms) | speedup |")
    print("|---|---|---|---|---|---|---|---|")
    sps = []
    for r in rows:
        sps.append(r[7] or float("nan"))
        print(f"| {r[0]} | {r[1]} | {r[2]:.4g} | {r[3]:.0f} | {r[4]:.3f} | {r[5]} | {r[6]} | "
              f"{(r[7] or float('nan')):.2f}x |")
    good = [x for x in sps if x == x]
    if good:
        print(f"\ngeomean speedup vs cuSPARSE best: "
              f"{math.exp(sum(math.log(x) for x in good) / len(good)):.2f}x over {len(good)} configs")


if __name__ == "__main__":
    main()
