"""Tensor-core precision versus pass count: eps = ||psi_gpu - psi_oracle||_2,
max |d psi| and |T - 1| at n = 24 (4x6, ABCDCDAB) for 20 / 40 / 80 cycles, tensor-core passes
(fuse_k 6) and CUDA-core fp32 passes (fuse_k 4) side by side.

    python scripts/precision_probe.py [--out profiles/r02_precision.txt]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--cycles", default="20,40,80")
    a = ap.parse_args()
    import oracle
    import paper_2512_07311_b200 as rcs
    from rcs_workload import emit_qasm, generate
    ctx = rcs.Context(0)
    lines = ["# n=24 (4x6 ABCDCDAB, seed 1): GPU vs fp64 oracle",
             "cycles  fuse_k  kernel  passes   eps=||dpsi||_2   max|dpsi|   T-1          oracle_s"]
    for cyc in [int(c) for c in a.cycles.split(",")]:
        text = emit_qasm(generate(4, 6, cyc, "ABCDCDAB", seed=1))
        t0 = time.time()
        ref = oracle.build_state(text)
        to = time.time() - t0
        c = rcs.Circuit.from_qasm(text)
        for k, kern in ((6, "auto"), (6, "k9"), (4, "auto")):
            st = rcs.State.build(ctx, c, fuse_k=k, tc_kernel=kern)
            psi = st.copy_out().astype(np.complex128)
            d = psi - ref
            lines.append(f"{cyc:6d}  {k:6d}  {kern:6s}  {st.report['n_passes']:6d}   {np.linalg.norm(d):.3e}        "
                         f"{np.abs(d).max():.3e}   {st.norm - 1:+.3e}   {to:.1f}")
            print(lines[-1], flush=True)
            st.free()
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
