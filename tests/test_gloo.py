"""World-size-2, 4 and 8 gloo tests of the N>1 host logic on CPU.

Each process holds one shard (top log2(P) qubits global) and executes the library's plan
(rcs_plan_create with n_global = log2 P): passes on local bits, REMAP items as a real
point-to-point exchange (pack the elements whose local swap bits equal the peer's code,
send/recv over gloo, unpack into the same positions -- the rule api.cpp implements with
NCCL), SWAP items locally.  Sampling uses the shard-total ownership rule of DESIGN.md §7
(E_r = sum of lower ranks' totals; the last rank with mass owns the tail).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def insert_zero_bits(m: np.ndarray, positions) -> np.ndarray:
    for s in sorted(positions):
        lo = m & ((1 << s) - 1)
        m = ((m >> s) << (s + 1)) | lo
    return m


def run_rank(rank, world, port, text, g, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2512_07311_b200 import Circuit, Plan
        from tests.plan_exec import apply_block, bit_swap
        c = Circuit.from_qasm(text)
        n = c.n_qubits
        nl = n - g
        plan = Plan(c, 4, g)
        items = plan.items()
        # product-state prefix (items [0, prefix): disjoint blocks on |0...0>, written by one
        # kernel on the GPU, possibly on global positions): every rank takes its slice of the
        # product state, built here on the full vector
        full0 = np.zeros(1 << n, np.complex128)
        full0[0] = 1
        for it in items[:plan.prefix]:
            assert it["type"] == "pass"
            apply_block(full0, it["matrix"], it["pos"])
        shard = full0[rank << nl:(rank + 1) << nl].copy()
        for it in items[plan.prefix:]:
            if it["type"] == "pass":
                assert max(it["pos"]) < nl
                apply_block(shard, it["matrix"], it["pos"])
            elif it["type"] == "swap":
                bit_swap(shard, list(zip(it["a"], it["b"])))
            else:
                j = it["k"]
                a, b = it["a"], it["b"]
                my = sum(((rank >> (a[i] - nl)) & 1) << i for i in range(j))
                m = np.arange(1 << (nl - j), dtype=np.int64)
                base = insert_zero_bits(m, b)
                reqs, bufs = [], {}
                for code in range(1 << j):
                    if code == my:
                        continue
                    peer = rank
                    mask = 0
                    for i in range(j):
                        gb = a[i] - nl
                        peer = (peer & ~(1 << gb)) | (((code >> i) & 1) << gb)
                        if (code >> i) & 1:
                            mask |= 1 << b[i]
                    idx = base | mask
                    send = torch.from_numpy(shard[idx].copy())
                    recv = torch.empty_like(send)
                    bufs[code] = (idx, recv)
                    reqs.append(dist.isend(send, peer))
                    reqs.append(dist.irecv(recv, peer))
                for r in reqs:
                    r.wait()
                for code, (idx, recv) in bufs.items():
                    shard[idx] = recv.numpy()
        # gather the state on rank 0
        t = torch.from_numpy(shard)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        full = torch.cat(parts).numpy()
        # sampling with shard ownership
        p = np.abs(shard) ** 2
        Tr = torch.tensor([p.sum()], dtype=torch.float64)
        tots = [torch.empty_like(Tr) for _ in range(world)]
        dist.all_gather(tots, Tr)
        tot = [float(x) for x in tots]
        E = float(np.sum(tot[:rank])) if rank else 0.0
        T = float(np.sum(tot))
        last = max(r for r in range(world) if tot[r] > 0)
        u = oracle.uniforms(2512, 20000)
        tt = u * T
        own = (tt >= E) & ((rank == last) | (tt < E + tot[rank])) & (tot[rank] > 0)
        C = np.cumsum(p)
        xs = np.searchsorted(C, tt - E, side="right")
        xs = np.minimum(xs, len(p) - 1) + (rank << nl)
        x = torch.from_numpy(np.where(own, xs, 0).astype(np.int64))
        dist.all_reduce(x)
        if rank == 0:
            q.put((full, x.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "c1"), (2, "grid"), (4, "grid"), (8, "grid16")])
def test_sharded_plan_over_gloo(world, case):
    import oracle
    from rcs_workload import config_qasm, emit_qasm, generate
    from paper_2512_07311_b200 import build
    build.build()
    text = {"c1": config_qasm("c1"), "grid": emit_qasm(generate(3, 5, 14, "ABCDCDAB", seed=7)),
            # world 8: g = 3 global qubits (7 peers per rank, j = 3 remaps), 4x4 grid
            "grid16": emit_qasm(generate(4, 4, 14, "ABCDCDAB", seed=9))}[case]
    g = world.bit_length() - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world + (7 if case != "c1" else 0)
    procs = [ctx.Process(target=run_rank, args=(r, world, port, text, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, x = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.build_state(text)
    assert np.abs(full - ref).max() < 1e-12
    u = oracle.uniforms(2512, 20000)
    xo, _ = oracle.sample(ref, u)
    C = np.cumsum(np.abs(ref) ** 2)
    t = u * C[-1]
    diff = np.nonzero(x.astype(np.uint64) != xo)[0]
    xg = x[diff]
    lo = np.where(xg > 0, C[np.maximum(xg - 1, 0)], 0.0) - 1e-6
    assert ((t[diff] >= lo) & (t[diff] <= C[xg] + 1e-6)).all()
