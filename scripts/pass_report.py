#!/usr/bin/env python
"""Per-pass timing report: kernel kind, target positions, ms, GB/s (run on the GPU box)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 6
c = rcs.Circuit.from_qasm(config_qasm(cfg))
n = c.n_qubits
ctx = rcs.Context(0)
plan = rcs.Plan(c, k, 0)
passes = [it for it in plan.items()[plan.prefix:] if it["type"] == "pass"]   # prefix blocks: no pass
st = None
for rep in range(3):
    if st is not None:
        amps, scratch = st.amps, st.scratch
        st.free()
        st = rcs.State.build(ctx, c, fuse_k=k, timing=True, amps=amps, scratch=scratch)
    else:
        st = rcs.State.build(ctx, c, fuse_k=k, timing=True)
t = st.pass_times()
rows = []
for it, ms in zip(passes, t):
    gbs = 16 * 2 ** n / (ms / 1e3) / 1e9
    rows.append((it["k"], sorted(it["pos"]), float(ms), gbs, it["n_gates"]))
    print(f"k={it['k']} pos={sorted(it['pos'])!s:28s} gates={it['n_gates']:3d} {ms:8.3f} ms {gbs:7.0f} GB/s")
print("build_ms", st.report["build_ms"], "sum pass ms", float(t.sum()))
json.dump([[a, b, float(c), float(d), e] for a, b, c, d, e in rows], open(f"gpurun_out/pass_report_{cfg}_k{k}.json", "w"))
