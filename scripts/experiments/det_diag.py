import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
ctx = rcs.Context(0)
text = emit_qasm(generate(3, 5, 4, 'ABCDCDAB', seed=0))
c = rcs.Circuit.from_qasm(text)
for g in (0, 2):
    ref = rcs.State.build(ctx, c, fuse_k=5, virtual_global=g).copy_out()
    diffs = []
    for rep in range(6):
        p = rcs.State.build(ctx, c, fuse_k=5, virtual_global=g).copy_out()
        diffs.append(int((p != ref).sum()))
    print("g", g, "repeat ndiffs", diffs)
# single padded-block circuit: product layer + one 5-qubit block region, g = 0 vs 2
text2 = emit_qasm(generate(3, 5, 2, 'ABCDCDAB', seed=0))
c2 = rcs.Circuit.from_qasm(text2)
a = rcs.State.build(ctx, c2, fuse_k=5).copy_out()
for g in (1, 2, 3):
    b = rcs.State.build(ctx, c2, fuse_k=5, virtual_global=g).copy_out()
    print("cyc2 g", g, "ndiff", int((a != b).sum()), [(i['type'], i['k'], i.get('pos', i.get('a'))) for i in rcs.Plan(c2, 5, g).items()])
