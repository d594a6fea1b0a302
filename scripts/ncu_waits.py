#!/usr/bin/env python
"""Where the warps of a tensor-core pass wait: warp-stall samples of an ncu --set full capture
(--page source --csv --print-source sass), attributed to the mbarrier each try_wait loop polls.

    python scripts/ncu_waits.py <sass.csv> [<raw.csv>]

Barrier offsets are K12's control block (tc_pass.cu k_pass_tct): rfull, rempty, afull, aempty,
dfull[2], dempty[2], cready[4] at 8-byte steps from the control base."""
import csv
import re
import sys

K12 = ["rfull[0]", "rfull[1]", "rempty[0]", "rempty[1]", "afull[0]", "afull[1]", "aempty[0]", "aempty[1]",
       "dfull[0]", "dfull[1]", "dempty[0]", "dempty[1]", "cready[0]", "cready[1]", "cready[2]", "cready[3]"]
ROLE = {"rfull": "converters wait for TMA data", "rempty": "producer waits for a free raw slot",
        "afull": "MMA waits for converted A", "aempty": "converters wait for a free A buffer",
        "dfull": "epilogue waits for the MMAs", "dempty": "MMA waits for the epilogue to read D",
        "cready": "epilogue waits for column exponents"}


def main(path, raw=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    total = sum(float(r[si] or 0) for r in data)
    base = None
    waits = {}
    for i, r in enumerate(data):
        m = re.search(r"TRYWAIT P(\d), \[(?:R\d+)?\+?URZ\+(0x[0-9a-f]+)\]", r[1])
        if not m:
            continue
        off = int(m.group(2), 16)
        for j in range(i + 1, min(i + 16, len(data))):   # the loop's back branch on that predicate
            if re.search(r"@!P%s\s+BRA" % m.group(1), data[j][1]):
                waits[off] = waits.get(off, 0.0) + float(data[j][si] or 0)
                break
    base = min(waits) if waits else 0
    print(f"{path}: {total:.0f} warp-stall samples")
    for off in sorted(waits):
        k = (off - base) // 8
        name = K12[k] if k < len(K12) else hex(off)
        role = ROLE.get(name.split("[")[0], "")
        print(f"  {name:10s} {waits[off]:10.0f}  {100 * waits[off] / total:5.1f} %  {role}")
    if raw:
        r = list(csv.reader(open(raw)))
        d = dict(zip(r[0], r[2]))
        for k in ("gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__inst_executed_op_tma_ld.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in d:
                print(f"  {k:75s} {d[k]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
