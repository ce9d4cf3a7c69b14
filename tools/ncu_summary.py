"""Summarise an `ncu --set full` report (.ncu-rep) per kernel launch into a text table for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]
Prints duration, DRAM bytes (read+write), registers, occupancy, IPC, FP64-pipe utilisation and
the top warp-stall reasons of every profiled launch.  With --json also writes a machine-readable
copy (bench.py reads `traffic` per kernel name from it when present).
"""
import csv
import json
import subprocess
import sys

KEYS = {
    "dur_ms": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_thru_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_thru_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}
UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
STALL = "smsp__average_warps_issue_stalled_"


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d["Kernel Name"].split("(")[0]}
        for k, m in KEYS.items():
            if m in d and d[m] != "":
                v = float(d[m].replace(",", ""))
                e[k] = v * UNIT.get(u[m], 1.0)
        stalls = {}
        for h in hdr:
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio") and d[h]:
                stalls[h[len(STALL):-len("_per_issue_active.ratio")]] = float(d[h])
        e["stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:4])
        e["traffic_bytes"] = (e.get("dram_rd_MB", 0) + e.get("dram_wr_MB", 0)) * 1e6
        res.append(e)
    return res


def main():
    rep = sys.argv[1]
    res = load(rep)
    print(f"# ncu --set full summary of {rep.split('/')[-1]} ({len(res)} launches)")
    print(f"{'kernel':34s} {'ms':>8s} {'DRAM MB':>8s} {'regs':>4s} {'grid':>7s} {'blk':>4s} "
          f"{'occ%':>5s} {'IPC':>5s} {'fp64%':>6s} {'SM%':>5s}  top stalls (cycles/issue)")
    for e in res:
        st = ", ".join(f"{k}={v:.2f}" for k, v in e["stalls"].items())
        print(f"{e['kernel'][:34]:34s} {e.get('dur_ms', 0):8.4f} "
              f"{e['traffic_bytes'] / 1e6:8.2f} {int(e.get('regs', 0)):4d} {int(e.get('grid', 0)):7d} "
              f"{int(e.get('block', 0)):4d} {e.get('warps_active_pct', 0):5.1f} {e.get('ipc', 0):5.2f} "
              f"{e.get('fp64_pipe_pct', 0):6.1f} {e.get('sm_thru_pct', 0):5.1f}  {st}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
