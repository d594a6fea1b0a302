"""Sustained power per pass kind: ~30-40 alternating 6-qubit blocks of one kind at n=34 (two
builds back to back, nvidia-smi sampled every 100 ms): pass ms, SM clock, board power."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from power_probe import sampler, stop
import torch
import paper_2512_07311_b200 as rcs

n = 34
KINDS = {
    "k9_rot_low0-5": ([0, 1, 2, 3, 4, 5], [0, 1, 2, 3, 4, 6]),
    "k9_low1_spread": ([2, 8, 14, 20, 26, 32], [2, 9, 15, 21, 27, 33]),
    "k9_low4-6": ([4, 5, 10, 11, 16, 22], [4, 6, 12, 13, 17, 23]),
    "k12_high": ([24, 25, 26, 27, 28, 29], [23, 24, 25, 26, 27, 28]),
    "k12_mid": ([7, 8, 9, 10, 11, 12], [8, 9, 10, 11, 12, 13]),
}


def qasm(Sa, Sb, layers=80):
    L = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{n}];"]
    for i in range(layers):
        S = Sa if i % 2 == 0 else Sb
        for q in S:
            L.append(f"sx q[{q}];")
        for a, b in zip(S[:-1], S[1:]):
            L.append(f"fsim(0.5,0.2) q[{a}],q[{b}];")
    return "\n".join(L) + "\n"


ctx = rcs.Context(0)
amps = torch.empty(1 << n, dtype=torch.complex64, device="cuda")
scratch = None
for name, (Sa, Sb) in KINDS.items():
    c = rcs.Circuit.from_qasm(qasm(Sa, Sb))
    st = rcs.State.build(ctx, c, fuse_k=6, amps=amps, scratch=scratch)
    scratch = st.scratch
    st.free()
    p, f = sampler()
    ms = []
    for _ in range(2):
        st = rcs.State.build(ctx, c, fuse_k=6, timing=True, amps=amps, scratch=scratch)
        ms += st.pass_times().tolist()
        st.free()
    sm, pw, tp = stop(p, f)
    last = ms[-20:]
    print(f"{name:16s} passes/build {len(ms) // 2:3d} ms first {ms[0]:.1f} median-last20 {statistics.median(last):.1f}"
          f" ({16 * 2 ** n / statistics.median(last) / 1e6:.0f} GB/s) | sm MHz median {statistics.median(sm):.0f}"
          f" | W median {statistics.median(pw):.0f} max {max(pw):.0f}", flush=True)
