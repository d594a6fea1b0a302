"""Pass kinds under the power cap on dense data: the C4 circuit (dense random state) followed by
~30 alternating 6-qubit blocks of one kind with varied gates (dense block matrices); reports the
appended passes' median time and the SM clock / board power over the whole build."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from power_probe import sampler, stop
import torch
import paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm

n = 34
KINDS = {
    "k9_rot_low0-5": ([0, 1, 2, 3, 4, 5], [0, 1, 2, 3, 4, 6]),
    "k9_low1_spread": ([2, 8, 14, 20, 26, 32], [2, 9, 15, 21, 27, 33]),
    "k9_low4-6": ([4, 5, 10, 11, 16, 22], [4, 6, 12, 13, 17, 23]),
    "k12_high": ([24, 25, 26, 27, 28, 29], [23, 24, 25, 26, 27, 28]),
    "k12_mid": ([7, 8, 9, 10, 11, 12], [8, 9, 10, 11, 12, 13]),
}
G1 = ["sx", "sy", "sw"]


def qasm(Sa, Sb, layers=80):
    base = config_qasm("c4").rstrip("\n").split("\n")
    L = list(base)
    for i in range(layers):
        S = Sa if i % 2 == 0 else Sb
        for j, q in enumerate(S):
            L.append(f"{G1[(i + j) % 3]} q[{q}];")
        for j, (a, b) in enumerate(zip(S[:-1], S[1:])):
            L.append(f"fsim({1.2 + 0.01 * ((i * 7 + j) % 31)},{0.3 + 0.01 * j}) q[{a}],q[{b}];")
    return "\n".join(L) + "\n"


ctx = rcs.Context(0)
amps = torch.empty(1 << n, dtype=torch.complex64, device="cuda")
scratch = None
base_passes = rcs.Plan(rcs.Circuit.from_qasm(config_qasm("c4")), 6, 0).n_passes
for name, (Sa, Sb) in KINDS.items():
    c = rcs.Circuit.from_qasm(qasm(Sa, Sb))
    st = rcs.State.build(ctx, c, fuse_k=6, amps=amps, scratch=scratch)
    scratch = st.scratch
    st.free()
    p, f = sampler()
    ms = []
    for _ in range(2):
        st = rcs.State.build(ctx, c, fuse_k=6, timing=True, amps=amps, scratch=scratch)
        t = st.pass_times().tolist()
        ms += t[base_passes + 2:]
        st.free()
    sm, pw, tp = stop(p, f)
    med = statistics.median(ms)
    print(f"{name:16s} appended passes {len(ms) // 2:3d} median {med:.1f} ms ({16 * 2 ** n / med / 1e6:.0f} GB/s)"
          f" | sm MHz median {statistics.median(sm):.0f} | W median {statistics.median(pw):.0f} max {max(pw):.0f}",
          flush=True)
