#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into small text/JSON files for profiles/.

    python scripts/summarize_ncu.py launches <launches.csv> <out.txt>   # per-kernel share of the step
    python scripts/summarize_ncu.py full <prof.ncu-rep> <out.txt>       # key --set full metrics
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot_t = 0.0
    for (i, name), m in per.items():
        short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        by[short][0] += 1
        by[short][1] += t
        by[short][2] += b
        tot_t += t
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary of {path}\n# kernel, launches, total ms, share of device time, "
                f"mean ms/launch, DRAM GB/launch, GB/s\n")
        for k, (n, t, b) in sorted(by.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:60s} {n:5d} {t / 1e6:10.3f} {t / tot_t:7.1%} {t / n / 1e6:9.3f} "
                    f"{b / n / 1e9:9.3f} {b / t if t else 0:8.1f}\n")
    print(open(out).read())


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {path}\n")
        for r in rows[2:]:
            f.write(f"kernel: {r[hdr.index('Kernel Name')]}\n")
            for m in FULL_METRICS:
                if m in hdr:
                    f.write(f"  {m:70s} {r[hdr.index(m)]:>16s} {units[hdr.index(m)]}\n")
    print(open(out).read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
