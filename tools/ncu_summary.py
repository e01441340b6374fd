"""Summarise an ncu --set full report (one kernel launch) into the numbers
DESIGN.md / bench.py cite: duration, DRAM bytes (the roofline "traffic"),
L2 / L1 throughput and hit rates, occupancy, registers, stall breakdown.

python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json] [--workload reddit]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sectors_srcunit_tex.sum": "l2_tex_sectors",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_l1_bytes",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_scoreboard",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg_throttle",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "stall_not_selected",
    "smsp__average_warp_latency_per_inst_issued.ratio": "cycles_per_issue",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                    u = "byte" if "byte" in u else "s"
                d[name] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
        if "l2_tex_sectors" in d and "duration" in d:
            d["l2_tex_TBps"] = d["l2_tex_sectors"] * 32 / d["duration"] / 1e12
        res.append(d)
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    r = summarize(rep)
    print(json.dumps(r, indent=1))
    if "--json" in sys.argv:
        json.dump(r, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
