import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
ctx = rcs.Context(0)
text = emit_qasm(generate(3, 5, 4, 'ABCDCDAB', seed=0))
c = rcs.Circuit.from_qasm(text)
a = rcs.State.build(ctx, c, fuse_k=5).copy_out()
for g in (2, 3):
    b = rcs.State.build(ctx, c, fuse_k=5, virtual_global=g).copy_out()
    print(os.environ.get("TAG", ""), "g", g, "ndiff", int((a != b).sum()))
