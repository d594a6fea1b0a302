"""torchrun worker for tests/test_multigpu.py: sharded build + sample + XEB over NCCL.

Each rank builds its shard through the C ABI, rank 0 gathers the state and compares it with
the single-GPU build (bitwise: the fusion plan is P-independent) and with the oracle; the
samples and XEB must equal the single-GPU results up to the G17 excuse band.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2512_07311_b200 as rcs
    from rcs_workload import SHOT_SEED

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = rcs.Context.from_process_group(local)
    results = {}
    opts = json.loads(os.environ.get("MGPU_OPTS", "{}"))
    from tests.test_multigpu import CASES
    for name, (text, k) in CASES.items():
        c = rcs.Circuit.from_qasm(text)
        n = c.n_qubits
        keep = name.endswith("_keep")
        st = rcs.State.build(ctx, c, fuse_k=k, timing=True, staging_bytes=1 << 20, keep_layout=keep, **opts)
        report = dict(st.report)
        x = st.sample(20000, seed=SHOT_SEED)
        xr = st.xeb(x)
        p = st.probabilities(x[:100])
        if keep:
            st.canonicalize()
        shard = torch.from_numpy(st.copy_out().view(np.float32).copy()).cuda()
        parts = [torch.empty_like(shard) for _ in range(world)]
        dist.all_gather(parts, shard)
        if rank == 0:
            full = torch.cat(parts).cpu().numpy().view(np.complex64)
            np.save(os.path.join(os.environ["MGPU_OUT"], f"{name}_state.npy"), full)
            np.save(os.path.join(os.environ["MGPU_OUT"], f"{name}_x.npy"), x)
            results[name] = {"n": n, "xeb": xr, "report": report, "p": p.tolist(), "norm": st.norm}
        st.free()
    if rank == 0:
        with open(os.path.join(os.environ["MGPU_OUT"], "results.json"), "w") as f:
            json.dump(results, f)
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
