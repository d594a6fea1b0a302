import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
shots = {"c3": 1_000_000, "c4": 2_500_000}[cfg]
ctx = rcs.Context(0)
c = rcs.Circuit.from_qasm(config_qasm(cfg))
n = c.n_qubits
t = time.perf_counter(); st = rcs.State.build(ctx, c, fuse_k=6); print("first build (plans) %.3f s" % (time.perf_counter() - t))
amps, scratch = st.amps, st.scratch
st.free()
x = torch.empty(shots, dtype=torch.int64, device="cuda")
for rep in range(3):
    t0 = time.perf_counter()
    st = rcs.State.build(ctx, c, fuse_k=6, timing=True, amps=amps, scratch=scratch)
    t1 = time.perf_counter()
    xs = st.sample(shots, device=True)
    t2 = time.perf_counter()
    r = st.xeb(xs)
    t3 = time.perf_counter()
    st.free()
    t4 = time.perf_counter()
    print(f"build wall {1e3*(t1-t0):.1f} ms (device {st.report['build_ms']:.1f}, plan {st.report['plan_ms']:.1f}) sample {1e3*(t2-t1):.1f} xeb {1e3*(t3-t2):.1f} free {1e3*(t4-t3):.1f}")
