#!/usr/bin/env python
"""Per-kernel SASS evidence of the tensor-core path: counts of the
tcgen05 / TMA mnemonics in every kernel of librcs.so (cuobjdump -sass, sm_100a).

    python scripts/sass_counts.py [--out profiles/r02/sass_counts.txt]
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2512_07311_b200", "librcs.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "FFMA", "FFMA2", "FMUL2",
       "FADD2", "F2FP", "FRND", "LDS", "STS", "LDG", "STG", "ATOMS", "PRMT"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m:
            counts[cur][m.group(1)] += 1
    lines = [f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)} (sm_100a): mnemonic counts per kernel",
             "kernel".ljust(60) + "".join(o.rjust(9) for o in OPS)]
    for fn, c in counts.items():
        short = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip() or fn
        short = re.sub(r"rcs::dev::\(anonymous namespace\)::", "", short)
        lines.append(short[:59].ljust(60) + "".join(str(c.get(o, 0)).rjust(9) for o in OPS))
    text = "\n".join(lines) + "\n"
    print(text, end="")
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
