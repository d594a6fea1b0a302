import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
ctx = rcs.Context(0)
text = emit_qasm(generate(3, 5, 4, 'ABCDCDAB', seed=0))
lines = text.splitlines()
head = [l for l in lines[:3]]
body = [l for l in lines[3:] if l and not l.startswith('barrier')]
for L in range(1, len(body) + 1):
    t = "\n".join(head + body[:L]) + "\n"
    c = rcs.Circuit.from_qasm(t)
    a = rcs.State.build(ctx, c, fuse_k=5).copy_out()
    b = rcs.State.build(ctx, c, fuse_k=5, virtual_global=2).copy_out()
    nd = int((a != b).sum())
    if nd:
        print("first divergent prefix", L, "ndiff", nd, "maxdiff %.3e" % np.abs(a - b).max())
        for g in (0, 2):
            for it in rcs.Plan(c, 5, g).items():
                print("  g", g, it['type'], it['k'], it.get('pos', it.get('a')), it.get('b', ''), it.get('qubits', ''), it.get('n_gates', ''))
        print("last gates:", body[max(0, L - 6):L])
        break
else:
    print("no divergence")
