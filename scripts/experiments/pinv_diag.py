import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
text = emit_qasm(generate(4, 5, 16, 'ABCDCDAB', seed=3))
ctx = rcs.Context(0)
s0 = rcs.State.build(ctx, rcs.Circuit.from_qasm(text), timing=True)
psi0 = s0.copy_out()
for g in (1, 2, 3):
    sg = rcs.State.build(ctx, rcs.Circuit.from_qasm(text), virtual_global=g, timing=True)
    p = sg.copy_out()
    d = np.abs(p - psi0)
    print(g, "ndiff", int((p != psi0).sum()), "maxdiff %.3e" % d.max(), "tc", sg.report["n_tc_passes"], "remaps", sg.report["n_remaps"], "swaps", sg.report["n_swaps"])
