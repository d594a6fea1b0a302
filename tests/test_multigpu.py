"""Real multi-GPU (NCCL over NVLink) parity: torchrun 2, 4 or 8 ranks vs single GPU and oracle.

Each world size skips when fewer GPUs are visible (gpurun --gpus 2/4 provides them; world 8
runs on a full 8-GPU box).  The NVLink data path is also covered on ONE GPU by the loopback
mode (tests/test_gpu_remap.py)."""
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


# name -> (qasm, fuse_k): k = 4 runs the CUDA-core passes with sequential remaps; k = 6 the
# tensor-core passes with remaps pipelined between them (n_pipelined > 0 in p2p modes)
CASES = {
    "c1": (config_qasm("c1"), 4),
    "grid20": (emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=3)), 4),
    "c2": (config_qasm("c2"), 4),
    "grid20_k6": (emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=3)), 6),
    "c2_k6": (config_qasm("c2"), 6),
    "grid26_k6": (emit_qasm(generate(2, 13, 14, "ABCD", seed=5)), 6),
    "c2_k6_keep": (config_qasm("c2"), 6),          # keep_layout: no final restore
}


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# build options per mode (rcs_build_opts): p2p = NVLink peer swaps pipelined with the neighbouring
# tensor-core passes (default: up to 3 passes after each remap); p2p_seq = not pipelined; p2p_c8 =
# 8 pipeline chunks, only the next pass behind the swaps; nccl =
# grouped send/recv remaps through the staging area
MODES = {"p2p": {}, "p2p_seq": {"overlap": False}, "p2p_c8": {"overlap_chunks": 3, "overlap_passes": 1},
         "nccl": {"remap_mode": "nccl"}}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_build_sample_xeb(world, mode, tmp_path, cuda_ok):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2512_07311_b200 import build
    build.build()
    env = dict(os.environ, MGPU_OUT=str(tmp_path), MGPU_OPTS=json.dumps(MODES[mode]))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + 10 * list(MODES).index(mode)),
                        os.path.join(ROOT, "tests", "mgpu_worker.py")], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.load(open(tmp_path / "results.json"))
    import paper_2512_07311_b200 as rcs
    ctx = rcs.Context(0)
    for name, (text, k) in CASES.items():
        full = np.load(tmp_path / f"{name}_state.npy")      # (keep cases: after canonicalize)
        single = rcs.State.build(ctx, rcs.Circuit.from_qasm(text), fuse_k=k)
        ref1 = single.copy_out()
        assert np.array_equal(full, ref1), name            # bitwise P-invariance
        ref = oracle.build_state(text)
        d = full.astype(np.complex128) - ref
        assert np.abs(d).max() <= 1e-5 and np.linalg.norm(d) <= 1e-5
        rep = res[name]["report"]
        assert rep["n_remaps"] > 0 or world == 1
        if k == 6 and mode in ("p2p", "p2p_c8"):
            assert rep["n_pipelined"] > 0, rep
        if mode in ("p2p_seq", "nccl") or k == 4:
            assert rep["n_pipelined"] == 0, rep
        assert rep["layout_kept"] == (1 if name.endswith("_keep") else 0), rep
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
