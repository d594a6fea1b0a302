"""bench.py host-side contract checks (no GPU)."""
import json
import subprocess
import sys

import pytest

from rcs_workload import CONFIGS, config_qasm


def test_plan_pass_table_matches_planner():
    import bench
    from paper_2512_07311_b200 import Circuit, Plan, build
    build.build()
    for cfg in CONFIGS:
        c = Circuit.from_qasm(config_qasm(cfg))
        for k in (3, 4, 5, 6):
            p = Plan(c, k, 0)
            assert bench.PLAN_PASSES[cfg][k] == p.n_passes, (cfg, k)
            assert bench.PLAN_PREFIX[cfg][k] == p.prefix, (cfg, k)
            if c.n_qubits >= 24:   # a function of the fused blocks, not of the sharding
                assert p.prefix == Plan(c, k, 2).prefix, (cfg, k)


def test_reference_arm_prints_one_json_line(tmp_path):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c2", "--steps", "1",
                        "--warmup", "0", "--cpu-budget", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == 1 and lines[0].startswith("{")
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
