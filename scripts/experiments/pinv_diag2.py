import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
text = emit_qasm(generate(4, 5, 16, 'ABCDCDAB', seed=3))
ctx = rcs.Context(0)
for k in (4, 5, 6):
    c = rcs.Circuit.from_qasm(text)
    psi0 = rcs.State.build(ctx, c, fuse_k=k).copy_out()
    for g in (1, 2, 3):
        p = rcs.State.build(ctx, c, fuse_k=k, virtual_global=g).copy_out()
        print("k", k, "g", g, "ndiff", int((p != psi0).sum()), "maxdiff %.3e" % np.abs(p - psi0).max(), flush=True)
