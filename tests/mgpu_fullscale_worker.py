"""torchrun worker for tests/test_multigpu_fullscale.py: the C5-size (n = 36) separable-circuit pin
on several GPUs (SURVEY §8.c.3 pin 2 at BASELINE north_star's target size).

C5's circuit with every coupler crossing grid rows 2|3 dropped factors as psi = psi_B (x) psi_A
(18 + 18 qubits, each from the fp64 oracle).  Every rank builds its shard (the state sharded on the
top log2(world) qubits, remaps over NVLink), compares it element by element on its device with
the matching rows of kron(psi_B, psi_A), and all ranks sample 2.5M shots and score XEB; rank 0
checks the shots against the exact two-level inverse CDF and writes results.json.
"""
import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

N, CUT, SHOTS = 36, 18, 2_500_000


def split_circuit():
    from rcs_workload import CONFIGS, emit_qasm, generate
    from rcs_workload.gen import Circuit as GenCircuit
    cfg = CONFIGS["c5"]
    full = generate(cfg["rows"], cfg["cols"], cfg["cycles"], cfg["pattern"], 1, n_qubits=N, jitter=0.05)
    cut, a, b = GenCircuit(N), GenCircuit(CUT), GenCircuit(N - CUT)
    dropped = 0
    for m in full.moments:
        keep, ma, mb = [], [], []
        for g in m:
            lo = [q < CUT for q in g.qubits]
            if all(lo):
                keep.append(g)
                ma.append(g)
            elif not any(lo):
                keep.append(g)
                mb.append(type(g)(g.kind, tuple(q - CUT for q in g.qubits), g.params))
            else:
                dropped += 1
        cut.moments.append(keep)
        a.moments.append(ma)
        b.moments.append(mb)
    assert dropped > 0
    return emit_qasm(cut), emit_qasm(a), emit_qasm(b)


def compare_kron(amps, f_hi, f_lo):
    """max |d| and sum |d|^2 of the device shard against kron(f_hi, f_lo), complex128, 2^26 at a time"""
    dev = amps.device
    lo = torch.from_numpy(np.ascontiguousarray(f_lo)).to(dev)
    hi = torch.from_numpy(np.ascontiguousarray(f_hi)).to(dev)
    nlo = lo.numel()
    rows = max(1, (1 << 26) // nlo)
    A = amps.view(-1, nlo)
    maxd, ss = 0.0, 0.0
    for r0 in range(0, hi.numel(), rows):
        d = A[r0:r0 + rows].to(torch.complex128) - hi[r0:r0 + rows, None] * lo[None, :]
        maxd = max(maxd, d.abs().max().item())
        ss += (d.real.square() + d.imag.square()).sum().item()
        del d
    return maxd, ss


def main():
    import oracle
    import paper_2512_07311_b200 as rcs
    from rcs_workload import SHOT_SEED

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = rcs.Context.from_process_group(local)
    text, qa, qb = split_circuit()
    psi_a, psi_b = oracle.build_state(qa), oracle.build_state(qb)
    g = world.bit_length() - 1
    st = rcs.State.build(ctx, rcs.Circuit.from_qasm(text), fuse_k=6)
    rep = dict(st.report)
    rows = 1 << (N - g - CUT)                     # psi_B rows of this rank's shard
    maxd, ss = compare_kron(st.amps, psi_b[rank * rows:(rank + 1) * rows], psi_a)
    x = st.sample(SHOTS, seed=SHOT_SEED)
    xr = st.xeb(x)
    norm = st.norm
    t = torch.tensor([maxd, ss], dtype=torch.float64, device="cuda")
    dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
    dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
    if rank == 0:
        maxd, eps = t[0].item(), math.sqrt(t[1].item())
        u = oracle.uniforms(SHOT_SEED, SHOTS)
        p_a, p_b = np.abs(psi_a) ** 2, np.abs(psi_b) ** 2
        CA, CB = np.cumsum(p_a), np.cumsum(p_b)
        TA, TB = CA[-1], CB[-1]
        tt = u * TA * TB
        xa = (x & np.uint64((1 << CUT) - 1)).astype(np.int64)
        xb = (x >> np.uint64(CUT)).astype(np.int64)
        CBm = np.where(xb > 0, CB[np.maximum(xb - 1, 0)], 0.0)
        CAm = np.where(xa > 0, CA[np.maximum(xa - 1, 0)], 0.0)
        hi = CBm * TA + p_b[xb] * CA[xa]
        lo = CBm * TA + p_b[xb] * CAm
        unexcused = int((~((tt >= lo - 1e-6) & (tt <= hi + 1e-6))).sum())
        F_exact = 2.0 ** N * np.mean(p_a[xa] * p_b[xb]) - 1
        fstar = (2.0 ** CUT * np.sum(p_a ** 2)) * (2.0 ** (N - CUT) * np.sum(p_b ** 2)) - 1
        res = {"world": world, "maxd": maxd, "eps": eps, "norm": norm, "unexcused": unexcused, "F": xr["F"],
               "sigma": xr["sigma"], "fstar_gpu": xr["fstar"], "F_exact": F_exact, "fstar": fstar, "report": rep}
        with open(os.path.join(os.environ["MGPU_OUT"], "fullscale.json"), "w") as f:
            json.dump(res, f)
        print(json.dumps({k: v for k, v in res.items() if k != "report"}))
    st.free()
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
