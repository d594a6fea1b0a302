"""Real multi-GPU (NCCL over NVLink) parity: torchrun 2 (or 4) ranks vs single GPU and oracle.

Skips when fewer than 2 GPUs are visible (gpurun --gpus 2 provides them)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from rcs_workload import SHOT_SEED, config_qasm, emit_qasm, generate

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("mode", ["p2p", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_build_sample_xeb(world, mode, tmp_path, cuda_ok):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2512_07311_b200 import build
    build.build()
    env = dict(os.environ, MGPU_OUT=str(tmp_path))
    if mode == "nccl":
        env["RCS_REMAP_NCCL"] = "1"   # grouped send/recv remaps instead of NVLink peer swaps
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + (10 if mode == "nccl" else 0)),
                        os.path.join(ROOT, "tests", "mgpu_worker.py")], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.load(open(tmp_path / "results.json"))
    import paper_2512_07311_b200 as rcs
    ctx = rcs.Context(0)
    texts = {"c1": config_qasm("c1"), "grid20": emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=3)),
             "c2": config_qasm("c2")}
    for name, text in texts.items():
        full = np.load(tmp_path / f"{name}_state.npy")
        single = rcs.State.build(ctx, rcs.Circuit.from_qasm(text), fuse_k=4)
        ref1 = single.copy_out()
        assert np.array_equal(full, ref1), name            # bitwise P-invariance
        ref = oracle.build_state(text)
        d = full.astype(np.complex128) - ref
        assert np.abs(d).max() <= 1e-5 and np.linalg.norm(d) <= 1e-5
        assert res[name]["report"]["n_remaps"] > 0 or world == 1
        x = np.load(tmp_path / f"{name}_x.npy")
        xs = single.sample(20000, seed=SHOT_SEED)
        u = oracle.uniforms(SHOT_SEED, 20000)
        C = np.cumsum(np.abs(ref) ** 2)
        t = u * C[-1]
        diff = np.nonzero(x != xs)[0]
        xg = x[diff].astype(np.int64)
        lo = np.where(xg > 0, C[np.maximum(xg - 1, 0)], 0.0) - 1e-6
        assert ((t[diff] >= lo) & (t[diff] <= C[xg] + 1e-6)).all(), name
        xr = res[name]["xeb"]
        F_o, _, _ = oracle.xeb(ref, x)
        assert abs(xr["F"] - F_o) <= 1e-3
        np.testing.assert_allclose(res[name]["p"], np.abs(ref[x[:100].astype(np.int64)]) ** 2, atol=1e-9)
        single.free()
