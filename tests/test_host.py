"""Host-side (no GPU) tests of the C-ABI library: symbol exports, the library's own QASM
parser against the oracle's, and the fused plan / remap planner via a NumPy executor."""
import math
import os
import re

import numpy as np
import pytest

import oracle
from rcs_workload import config_qasm, emit_qasm, generate, random_qasm
from tests.plan_exec import run_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rcs():
    from paper_2512_07311_b200 import build
    build.build()
    import paper_2512_07311_b200 as m
    return m


def test_library_exports_every_header_symbol(rcs):
    hdr = open(os.path.join(ROOT, "include", "rcs.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(rcs_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 20
    L = rcs.lib()
    for nm in sorted(names):
        assert hasattr(L, nm), nm
    from paper_2512_07311_b200._lib import SIGNATURES
    assert names == set(SIGNATURES), names ^ set(SIGNATURES)
    assert L.rcs_status_string(6) == b"RCS_ERR_NORM"


def _lib_gates(rcs, text):
    return rcs.Circuit.from_qasm(text).gates()


@pytest.mark.parametrize("src", ["c1", "c2", "c3", "c4", "c5", "rand0", "rand1", "rand2", "meas"])
def test_parser_matches_oracle_parser(rcs, src):
    if src.startswith("rand"):
        text = random_qasm(7, 120, int(src[4:]))
    elif src == "meas":
        text = emit_qasm(generate(2, 3, 4, "ABCD", 9), measure=True)
    else:
        text = config_qasm(src)
    o = oracle.parse(text)
    c = rcs.Circuit.from_qasm(text)
    st = c.stats()
    assert st["n_qubits"] == o.n_qubits and st["n_moments"] == o.n_moments and st["n_measure"] == o.n_measure
    lg = c.gates()
    assert len(lg) == len(o.gates)
    for (k, qs, th, ph, m), g in zip(lg, o.gates):
        assert (k, qs, m) == (g.kind, g.qubits, g.moment)
        assert th == g.theta and ph == g.phi          # bit-identical angle parsing


@pytest.mark.parametrize("text", [
    "OPENQASM 2.0;\nqreg q[2];\nfoo q[0];\n",
    "OPENQASM 2.0;\nqreg q[2];\nsx q[2];\n",
    "OPENQASM 2.0;\nqreg q[2];\nfsim(0.1) q[0],q[1];\n",
    "OPENQASM 2.0;\nqreg q[2];\nsx q[0],q[1];\n",
    "OPENQASM 2.0;\nqreg q[2];\nfsim(1,2) q[1],q[1];\n",
    "OPENQASM 2.0;\nqreg q[2];\n  sx q[0]\n",
    "OPENQASM 2.0;\nsx q[0];\n",
    "OPENQASM 2.0;\nqreg q[3];\nrz(pi*) q[0];\n",
])
def test_parser_errors_match_oracle(rcs, text):
    with pytest.raises(oracle.OracleError) as eo:
        oracle.parse(text)
    with pytest.raises(rcs.RcsError) as el:
        rcs.Circuit.from_qasm(text)
    assert el.value.status == "RCS_ERR_" + eo.value.name
    assert (el.value.line, el.value.col) == (eo.value.line, eo.value.col)


def test_block_matrices_unitary_and_cover_all_gates(rcs):
    c = rcs.Circuit.from_qasm(config_qasm("c2"))
    for k in (2, 3, 4, 5, 6):
        p = rcs.Plan(c, k, 0)
        items = p.items()
        tot = 0
        for it in items:
            assert it["type"] == "pass" and 1 <= it["k"] <= k
            M = it["matrix"]
            assert np.abs(M.conj().T @ M - np.eye(M.shape[0])).max() < 1e-12
            assert it["qubits"] == sorted(it["qubits"]) and it["pos"] == it["qubits"]
            tot += it["n_gates"]
        assert tot == c.stats()["n_gates"]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_plan_executor_matches_oracle_random(rcs, seed, k):
    n = 4 + seed % 6 if k < 6 else 12 + seed % 3
    text = random_qasm(n, 60, 1000 + seed)
    ref = oracle.build_state(text)
    c = rcs.Circuit.from_qasm(text)
    p = rcs.Plan(c, k, 0)
    psi = run_plan(p.items(), n)
    assert np.abs(psi - ref).max() < 1e-12


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("grid", [(3, 4, 14, "EFGH"), (2, 6, 20, "ABCDCDAB"), (3, 5, 12, "ABCD")])
def test_plan_with_global_qubits_restores_canonical_order(rcs, g, grid):
    rows, cols, cyc, pat = grid
    n = rows * cols
    if n - g - 7 < (6 if n - g >= 12 else 4):
        pytest.skip("too few movable local qubits (positions 0..5 are pinned)")
    text = emit_qasm(generate(rows, cols, cyc, pat, seed=g))
    ref = oracle.build_state(text)
    c = rcs.Circuit.from_qasm(text)
    p = rcs.Plan(c, 6 if n - g >= 12 else 4, g)
    items = p.items()
    nl = n - g
    for i, it in enumerate(items):
        if i < p.prefix:   # product-state prefix blocks: written by one kernel, any position
            continue
        if it["type"] == "pass":
            assert max(it["pos"]) < nl                          # blocks only touch local bits
        elif it["type"] == "remap":
            assert all(a >= nl for a in it["a"]) and all(6 <= b < nl for b in it["b"])
        else:
            assert all(6 <= a < nl and 6 <= b < nl for a, b in zip(it["a"], it["b"]))
    # the fusion is independent of the number of global qubits (P-invariance)
    p0 = rcs.Plan(c, 6 if n - g >= 12 else 4, 0)
    b0 = [i for i in p0.items() if i["type"] == "pass"]
    bg = [i for i in items if i["type"] == "pass"]
    assert len(b0) == len(bg)
    for x, y in zip(b0, bg):
        assert x["qubits"] == y["qubits"] and np.array_equal(x["matrix"], y["matrix"])
    psi = run_plan(items, n)
    assert np.abs(psi - ref).max() < 1e-12


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("grid", [(3, 5, 14, "EFGH"), (2, 8, 20, "ABCDCDAB"), (4, 4, 12, "ABCD")])
def test_kept_layout_plan(rcs, g, grid):
    """keep_layout executes items [0, restore_begin): the physical state then equals the oracle
    state with qubit q moved to final_pos[q] (pins the layout the logical CDF relies on)."""
    rows, cols, cyc, pat = grid
    n = rows * cols
    if n - g - 7 < (6 if n - g >= 12 else 4):
        pytest.skip("too few movable local qubits")
    text = emit_qasm(generate(rows, cols, cyc, pat, seed=20 + g))
    ref = oracle.build_state(text)
    c = rcs.Circuit.from_qasm(text)
    p = rcs.Plan(c, 6 if n - g >= 12 else 4, g)
    lay = p.layout()
    items = p.items()
    assert all(it["type"] == "pass" for it in items[:lay["restore_begin"]][-1:])
    assert all(it["type"] != "pass" for it in items[lay["restore_begin"]:])
    assert sorted(lay["final_pos"]) == list(range(n)) and sorted(lay["initial_pos"]) == list(range(n))
    assert all(lay["final_pos"][q] == q for q in range(6))           # positions 0..5 pinned
    psi = run_plan(items[:lay["restore_begin"]], n)
    # physical index of logical x: bit q of x goes to position final_pos[q]
    x = np.arange(1 << n, dtype=np.int64)
    phys = np.zeros_like(x)
    for q in range(n):
        phys |= ((x >> q) & 1) << lay["final_pos"][q]
    assert np.abs(psi[phys] - ref).max() < 1e-12
    assert np.abs(run_plan(items, n) - ref).max() < 1e-12             # with the restore: canonical


def test_plan_rejects_bad_arguments(rcs):
    c = rcs.Circuit.from_qasm(config_qasm("c1"))
    with pytest.raises(rcs.RcsError):
        rcs.Plan(c, 7, 0)
    with pytest.raises(rcs.RcsError):
        rcs.Plan(c, 4, 3)   # 12 - 3 - 6 < 4 movable local qubits


def test_pass_counts_reported(rcs):
    # fusion quality guard: k=4 passes for the BASELINE configs
    want = {"c1": 22, "c2": 52, "c3": 68, "c4": 86, "c5": 93}
    for cfg, cap in want.items():
        p = rcs.Plan(rcs.Circuit.from_qasm(config_qasm(cfg)), 4, 0)
        assert p.n_passes <= cap, (cfg, p.n_passes)


def key_of(p):
    return [tuple((f, np.asarray(v).tobytes()) for f, v in sorted(it.items())) for it in p.items()]


def test_plan_deterministic_across_runs(rcs):
    """The fusion strategies run in threads and share a memo of greedy rollouts:
    the plan must not depend on thread timing -- the same items, run after run."""
    c = rcs.Circuit.from_qasm(config_qasm("c2"))
    runs = [key_of(rcs.Plan(c, 6, g)) for g in (0, 0, 0, 2, 2)]
    assert runs[0] == runs[1] == runs[2]
    assert runs[3] == runs[4]


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_plan_deterministic_all_widths(rcs, cfg):
    """Every block width, fresh circuit objects each run (no per-circuit plan cache): identical
    items and matrices.  A memo shared between strategies with different rollout functions once
    made C4's k = 5 plan vary between runs (56 / 57 passes); this would catch it."""
    text = config_qasm(cfg)
    for k in (4, 5, 6):
        runs = [key_of(rcs.Plan(rcs.Circuit.from_qasm(text), k, 0)) for _ in range(3)]
        assert runs[0] == runs[1] == runs[2], (cfg, k)
