"""C5-size oracle-anchored parity on several GPUs (BASELINE north_star: "C5 n=36 ... matching the
oracle"): the separable-circuit pin (SURVEY §8.c.3 pin 2) at n = 36, state sharded over 4 or 8
GPUs with NVLink remaps.  PAPER.md §3.2 l.36 (stage 1 constructs the complete state), SPEC.md:130,
:152 (equal to the reference state).  Tolerances as tests/test_gpu_fullscale.py: max |d psi| and
||d psi||_2 <= 1e-5 (G16), 2.5M shots within G17, same-sample XEB within 1e-3, F* within 1e-4."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [4, 8])
def test_separable_c5_n36_sharded(world, tmp_path, cuda_ok):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2512_07311_b200 import build
    build.build()
    env = dict(os.environ, MGPU_OUT=str(tmp_path))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29700 + world),
                        os.path.join(ROOT, "tests", "mgpu_fullscale_worker.py")], env=env, capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.load(open(tmp_path / "fullscale.json"))
    print(json.dumps({k: v for k, v in res.items() if k != "report"}))
    assert res["report"]["n_remaps"] > 0 and res["report"]["n_tc_passes"] > 0, res["report"]
    assert res["maxd"] <= 1e-5 and res["eps"] <= 1e-5, res
    assert abs(res["norm"] - 1) <= 1e-5
    assert res["unexcused"] == 0, res
    assert abs(res["F"] - res["F_exact"]) <= 1e-3, res
    assert abs(res["fstar_gpu"] - res["fstar"]) <= 1e-4, res
