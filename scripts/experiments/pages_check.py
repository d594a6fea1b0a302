"""Single 6-qubit pass timing vs target positions (how many targets sit above the 2 MB page,
amplitude bit 18): one circuit per position set, one tensor-core pass each, K12 and K9."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2512_07311_b200 as rcs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
SETS = [[0, 1, 2, 3, 4, 5], [7, 8, 9, 10, 11, 12], [12, 13, 14, 15, 16, 17], [14, 15, 16, 17, 18, 19],
        [16, 17, 18, 19, 20, 21], [17, 18, 19, 20, 21, 22], [18, 19, 20, 21, 22, 23], [24, 25, 26, 27, 28, 29],
        [n - 6, n - 5, n - 4, n - 3, n - 2, n - 1], [7, 8, 9, 30, 31, 32], [7, 8, 26, 27, 31, 32],
        [2, 8, 14, 20, 26, 32], [13, 19, 25, 26, 31, 32], [11, 17, 23, 24, 28, 29]]


def qasm(S):
    L = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{n}];"]
    for rep in range(2):
        for q in S:
            L.append(f"sx q[{q}];")
        for a, b in zip(S[:-1], S[1:]):
            L.append(f"fsim(0.5,0.2) q[{a}],q[{b}];")
    return "\n".join(L) + "\n"


ctx = rcs.Context(0)
amps = scratch = None
for S in SETS:
    if max(S) >= n:
        continue
    c = rcs.Circuit.from_qasm(qasm(S))
    hp = sum(1 for q in S if q >= 18)
    res = []
    for mode in ("k12", "k9"):
        if mode == "k9":
            os.environ["RCS_TC_NOTRANS"] = "1"
        else:
            os.environ.pop("RCS_TC_NOTRANS", None)
        ts = []
        for rep in range(4):
            st = rcs.State.build(ctx, c, fuse_k=6, timing=True, amps=amps, scratch=scratch)
            amps, scratch = st.amps, st.scratch
            t = st.pass_times()
            ts.append(float(t.max()))
            npass = len(t)
            st.free()
        ms = min(ts[1:])
        res.append(f"{mode} {ms:7.2f} ms {16 * 2 ** n / ms / 1e6:6.0f} GB/s")
    print(f"S={S!s:32s} page-bits={hp} passes={npass}  " + "  ".join(res), flush=True)
