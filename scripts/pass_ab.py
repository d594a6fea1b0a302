#!/usr/bin/env python
"""Per-pass times of one circuit under two tensor-core kernel choices (auto vs K9 for every block,
or vs another tc_kernel mode), alternating on one GPU:
    python scripts/pass_ab.py rows cols cycles pattern [seed] [other mode: k9 | norow]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07311_b200 as rcs  # noqa: E402
from rcs_workload import emit_qasm, generate  # noqa: E402

rows, cols, cyc, pat = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 1
other = sys.argv[6] if len(sys.argv) > 6 else "k9"
c = rcs.Circuit.from_qasm(emit_qasm(generate(rows, cols, cyc, pat, seed=seed)))
ctx = rcs.Context(0)
plan = rcs.Plan(c, 6, 0)
passes = [it for it in plan.items()[plan.prefix:] if it["type"] == "pass"]
res = {}
st = None
for rep in range(2):
    for kern in ("auto", other):
        kw = dict(fuse_k=6, timing=True, tc_kernel=kern)
        if st is not None:
            kw.update(amps=st.amps, scratch=st.scratch)
            st.free()
        st = rcs.State.build(ctx, c, **kw)
        res[kern] = st.pass_times()
for it, a, b in zip(passes, res["auto"], res[other]):
    low = sum(p < 4 for p in it["pos"])
    print(f"pos={it['pos']!s:28s} low={low}  auto {a:8.3f} ms  {other} {b:8.3f} ms")
