import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import emit_qasm, generate
ctx = rcs.Context(0)
found = 0
for rows, cols, cyc in [(3, 5, 2), (3, 5, 3), (3, 5, 4), (4, 4, 3), (4, 4, 5), (4, 5, 3), (4, 5, 6)]:
    for seed in range(4):
        text = emit_qasm(generate(rows, cols, cyc, 'ABCDCDAB', seed=seed))
        c = rcs.Circuit.from_qasm(text)
        n = c.n_qubits
        psi0 = rcs.State.build(ctx, c, fuse_k=5).copy_out()
        for g in (1, 2, 3):
            if n - g < 12:
                continue
            p = rcs.State.build(ctx, c, fuse_k=5, virtual_global=g).copy_out()
            nd = int((p != psi0).sum())
            if nd:
                print(f"DIFF n={n} cyc={cyc} seed={seed} g={g} ndiff={nd} maxdiff={np.abs(p - psi0).max():.3e}")
                if found < 2:
                    for gg in (0, g):
                        pl = rcs.Plan(c, 5, gg)
                        print("  plan g", gg, [(i['type'], i['k'], i.get('pos', i.get('a')), i.get('b')) for i in pl.items()])
                found += 1
print("done, found", found)
