"""Pins of the fp64 CPU oracle against things other than itself (no GPU needed).

Every pin names what fixes it: SPEC.md worked examples (tests/golden/), closed forms,
invariants, textbook routines (dense unitary products, numpy cumsum/searchsorted, the
published SplitMix64 vector) or statistics.  A plausible mistake in the oracle (wrong
matrix entry or sign, transposed operand, wrong bit order, dropped term, off-by-one CDF)
fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from rcs_workload import config_qasm, generate, emit_qasm, random_qasm
from tests.dense_unitary import dense_state, embed, kron_1q

GOLD = os.path.join(os.path.dirname(__file__), "golden")
X = np.array([[0, 1], [1, 0]], dtype=complex)
Y = np.array([[0, -1j], [1j, 0]], dtype=complex)
W = (X + Y) / math.sqrt(2)


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- O2 matrices
def test_sqrtx_matches_spec_example():
    g = gold("spec_examples.json")["sqrtx_matrix"]
    M = oracle.gate_matrix("sx")
    np.testing.assert_allclose(M, np.array(g["re"]) + 1j * np.array(g["im"]), atol=1e-15)


@pytest.mark.parametrize("kind,U", [("sx", X), ("sy", Y), ("sw", W)])
def test_square_roots_square_to_U(kind, U):
    # M.M = U  (principal square roots, reading V2)
    M = oracle.gate_matrix(kind)
    assert np.abs(M @ M - U).max() <= 1e-12
    # principal root: eigenvalues of sqrt(U) are 1 and i (arguments in (-pi/2, pi/2])
    ev = np.sort_complex(np.linalg.eigvals(M))
    np.testing.assert_allclose(sorted(ev, key=lambda z: z.imag), [1, 1j], atol=1e-12)


@pytest.mark.parametrize("kind,th,ph", [("sx", 0, 0), ("sy", 0, 0), ("sw", 0, 0), ("rz", 0, 0.7),
                                        ("rz", 0, -2.1), ("fsim", 1.1, 0.3), ("fsim", -0.4, 2.5),
                                        ("fsim", math.pi / 2, math.pi / 6)])
def test_unitarity(kind, th, ph):
    M = oracle.gate_matrix(kind, th, ph)
    assert np.abs(M.conj().T @ M - np.eye(M.shape[0])).max() <= 1e-12


def test_fsim_closed_forms():
    th, ph = 0.83, 0.37
    M = oracle.gate_matrix("fsim", th, ph)
    e = np.eye(4)
    # fSim |11> = e^{-i phi} |11>
    np.testing.assert_allclose(M @ e[3], np.exp(-1j * ph) * e[3], atol=1e-15)
    # |00> unchanged
    np.testing.assert_allclose(M @ e[0], e[0], atol=1e-15)
    # fSim(0, 0) = I
    np.testing.assert_allclose(oracle.gate_matrix("fsim", 0, 0), np.eye(4), atol=1e-15)
    # fSim(pi/2, phi) = SWAP . diag(1, -i, -i, e^{-i phi})  (closed form)
    SWAP = np.eye(4)[[0, 2, 1, 3]]
    np.testing.assert_allclose(oracle.gate_matrix("fsim", math.pi / 2, ph),
                               SWAP @ np.diag([1, -1j, -1j, np.exp(-1j * ph)]), atol=1e-15)
    # the |01>,|10> block is exp(-i theta X): generator check via the derivative at 0
    d = (oracle.gate_matrix("fsim", 1e-6, 0) - oracle.gate_matrix("fsim", -1e-6, 0)) / 2e-6
    np.testing.assert_allclose(d[1:3, 1:3], -1j * X, atol=1e-9)


def test_rz_is_phase_on_basis_states():
    # Rz on a basis state keeps it up to phase; relative phase e^{i phi}
    ph = 0.91
    M = oracle.gate_matrix("rz", 0, ph)
    assert abs(M[0, 1]) == 0 and abs(M[1, 0]) == 0
    assert abs(M[1, 1] / M[0, 0] - np.exp(1j * ph)) < 1e-15
    assert abs(abs(M[0, 0]) - 1) < 1e-15


# ---------------------------------------------------------------- O3/O4 evolution
def test_spec_worked_examples():
    g = gold("spec_examples.json")
    e = g["empty_circuit_n3"]
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[3];\n")
    np.testing.assert_array_equal(psi, np.array(e["re"]) + 1j * np.array(e["im"]))
    s = g["sqrtx_on_zero"]
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[1];\nx_1_2 q[0];\n")
    np.testing.assert_allclose(psi, np.array(s["re"]) + 1j * np.array(s["im"]), atol=1e-16)


def test_bit_order_qubit0_is_lsb():
    # index i has qubit q as bit q.  sqrt(X) twice = X flips the qubit.
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[3];\nsx q[1];\nsx q[1];\n")
    assert abs(abs(psi[0b010]) - 1) < 1e-15


@pytest.mark.parametrize("seed", range(200))
def test_random_circuits_vs_dense_unitary(seed):
    # SPEC S:152 / acceptance 1: n <= 6, up to 12 cycles, 1e-10 max deviation
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 7))
    text = random_qasm(n, int(rng.integers(0, 40)), seed)
    c = oracle.parse(text)
    psi = c.build_state()
    ref = dense_state(c.gates, n, oracle.gate_matrix)
    assert np.abs(psi - ref).max() <= 1e-10


@pytest.mark.parametrize("rows,cols,cycles,pat", [(2, 3, 8, "ABCDCDAB"), (3, 3, 6, "EFGH"), (2, 4, 10, "ABCD")])
def test_grid_circuits_vs_dense_unitary(rows, cols, cycles, pat):
    circ = generate(rows, cols, cycles, pat, seed=5)
    c = oracle.parse(emit_qasm(circ))
    n = rows * cols
    psi = c.build_state()
    ref = dense_state(c.gates, n, oracle.gate_matrix)
    assert np.abs(psi - ref).max() <= 1e-10


def test_kron_embedding_agrees_for_1q():
    # two structurally different embeddings of 1q gates agree (pins the dense checker too)
    for q in range(4):
        M = oracle.gate_matrix("sw")
        np.testing.assert_allclose(embed(M, (q,), 4), kron_1q(M, q, 4), atol=0)


def test_two_qubit_operand_order():
    # basis index b_q0 + 2 b_q1: a non-symmetric probe -- apply fSim on (0, 2)
    # to |q0=1> and check the -i sin(theta) amplitude lands on |q1=1>
    th = 0.3
    psi = np.zeros(8, complex)
    psi[0b001] = 1
    oracle.apply_gate(psi, "fsim", (0, 2), th, 0.0)
    np.testing.assert_allclose(psi[0b001], math.cos(th), atol=1e-16)
    np.testing.assert_allclose(psi[0b100], -1j * math.sin(th), atol=1e-16)


def test_disjoint_gates_commute_and_determinism():
    # SPEC S:153-154
    rng = np.random.default_rng(1)
    psi0 = rng.normal(size=64) + 1j * rng.normal(size=64)
    psi0 /= np.linalg.norm(psi0)
    a, b = psi0.copy(), psi0.copy()
    oracle.apply_gate(a, "sw", (1,)); oracle.apply_gate(a, "fsim", (3, 5), 0.4, 0.9)
    oracle.apply_gate(b, "fsim", (3, 5), 0.4, 0.9); oracle.apply_gate(b, "sw", (1,))
    assert np.abs(a - b).max() <= 1e-12
    t = config_qasm("c1")
    s1, s2 = oracle.build_state(t), oracle.build_state(t)
    assert s1.tobytes() == s2.tobytes()


def test_norm_preserved():
    # SPEC S:113
    psi = oracle.build_state(config_qasm("c1"))
    assert abs(oracle.total_prob(psi) - 1) <= 1e-12 * 227


def test_product_state_closed_form():
    # 1q-only circuit: psi_x = prod_q v_q[x_q]  (SURVEY §8.c.3 full-scale pin 1)
    circ = generate(4, 4, 6, "ABCD", seed=3, two_qubit=False)
    c = oracle.parse(emit_qasm(circ))
    psi = c.build_state()
    n = 16
    v = [np.array([1, 0], complex) for _ in range(n)]
    for g in c.gates:
        v[g.qubits[0]] = oracle.gate_matrix(g.kind) @ v[g.qubits[0]]
    ref = v[n - 1]
    for q in range(n - 2, -1, -1):
        ref = np.kron(ref, v[q])
    assert np.abs(psi - ref).max() <= 1e-14


def inverse_qasm(c):
    """C^dagger: reversed order; sqrt(U)^dagger = sqrt(U)^3; fSim(t,p)^dagger = fSim(-t,-p)."""
    names = {"sx": "x_1_2", "sy": "y_1_2", "sw": "hz_1_2"}
    lines = []
    for g in reversed(c.gates):
        if g.kind in names:
            lines += [f"{names[g.kind]} q[{g.qubits[0]}];"] * 3
        elif g.kind == "rz":
            lines.append(f"rz({-g.phi!r}) q[{g.qubits[0]}];")
        else:
            lines.append(f"fsim({-g.theta!r},{-g.phi!r}) q[{g.qubits[0]}],q[{g.qubits[1]}];")
    return "\n".join(lines) + "\n"


def test_circuit_then_inverse_is_identity():
    t = config_qasm("c1")
    c = oracle.parse(t)
    both = oracle.parse(t + inverse_qasm(c))
    psi = both.build_state()
    assert abs(psi[0] - 1) <= 1e-12 and np.abs(psi[1:]).max() <= 1e-12


# ---------------------------------------------------------------- O7 uniforms
def test_uniforms_splitmix_vector():
    g = gold("splitmix64.json")
    u = oracle.uniforms(g["seed"], 3)
    expect = [(int(h, 16) >> 11) * 2.0 ** -53 for h in g["outputs_hex"]]
    assert list(u) == expect
    # counter-based: offset windows agree with the full stream
    full = oracle.uniforms(2512, 1000)
    np.testing.assert_array_equal(oracle.uniforms(2512, 100, offset=400), full[400:500])
    big = oracle.uniforms(7, 200000)
    assert big.min() >= 0 and big.max() < 1 and abs(big.mean() - 0.5) < 0.005


# ---------------------------------------------------------------- O8 sampling
def brute_inverse_cdf(psi, u):
    p = np.abs(psi) ** 2
    C = np.cumsum(p)                        # sequential fp64 cumulative sum
    T = C[-1]
    x = np.searchsorted(C, u * T, side="right")
    last = np.nonzero(p > 0)[0][-1]
    return np.where(x >= len(p), last, x).astype(np.uint64)


@pytest.mark.parametrize("n,seed", [(1, 0), (3, 1), (6, 2), (8, 3), (10, 4)])
def test_sampler_equals_brute_force_inverse_cdf(n, seed):
    text = random_qasm(n, 6 * n, seed)
    psi = oracle.build_state(text)
    u = oracle.uniforms(2512 + seed, 20000)
    x, T = oracle.sample(psi, u)
    np.testing.assert_array_equal(x, brute_inverse_cdf(psi, u))


def test_sampler_point_mass_and_binomial():
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[4];\n")
    x, _ = oracle.sample(psi, oracle.uniforms(1, 1000))
    assert (x == 0).all()
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[1];\nsx q[0];\n")
    S = 100000
    x, _ = oracle.sample(psi, oracle.uniforms(2, S))
    assert abs((x == 0).mean() - 0.5) <= 4 * math.sqrt(0.25 / S)


def test_sampler_chi_square_and_tv():
    from scipy.stats import chi2
    text = emit_qasm(generate(2, 3, 10, "ABCDCDAB", seed=11))
    psi = oracle.build_state(text)
    p = np.abs(psi) ** 2
    S = 200000
    x, _ = oracle.sample(psi, oracle.uniforms(3, S))
    cnt = np.bincount(x.astype(np.int64), minlength=64)
    stat = ((cnt - S * p) ** 2 / (S * p)).sum()
    assert stat < chi2.ppf(0.999, 63)
    tv = 0.5 * np.abs(cnt / S - p).sum()
    assert tv <= 3 * math.sqrt(64 / S)


def test_inverse_cdf_ties_and_zero_probabilities():
    """V13 on hand-computed cases: x_s = min{x : C(x) > t_s} with C the INCLUSIVE
    CDF, so a t_s that lands exactly on C(x) picks the next x with p > 0 (a `>=` comparison
    would pick x itself, or a zero-probability x)."""
    psi = np.zeros(8, complex)
    psi[0], psi[2], psi[3] = 0.5, 0.5, 0.5 + 0.5j       # p = [1/4, 0, 1/4, 1/2, 0, 0, 0, 0] exactly
    u = np.array([0.0, 0.2, 0.25, 0.4, 0.5, 0.75, 1 - 2.0 ** -53])
    x, T = oracle.sample(psi, u)
    assert T == 1.0
    assert x.tolist() == [0, 0, 2, 2, 3, 3, 3]


def test_inverse_cdf_fallback_is_last_nonzero():
    """V13's fallback: when no x has C(x) > t_s, the pick is the last x WITH p > 0 -- not the last
    index 2^n - 1 (a plain searchsorted would return 2^n and clip to a zero-probability index).
    The oracle's T is the CDF's own end C(2^n - 1), so fl(u T) < T for every u < 1 and the branch
    is reached through the uniform hook with u = 1 (t = T), on states with trailing zeros."""
    psi = np.zeros(8, complex)
    psi[0], psi[2], psi[3] = 0.5, 0.5, 0.5 + 0.5j       # p = [1/4, 0, 1/4, 1/2, 0, 0, 0, 0]
    x, T = oracle.sample(psi, np.array([1.0, 1 - 2.0 ** -53]))
    assert x.tolist() == [3, 3]
    psi = np.zeros(16, complex)
    psi[[1, 4, 5]] = [0.5, 0.5j, 0.5 + 0.5j]             # p = 1/4, 1/4, 1/2; last non-zero at 5
    x, T = oracle.sample(psi, np.array([1.0, 0.0, 0.25, 0.5]))
    assert x.tolist() == [5, 1, 4, 5]
    # fl(u T) < T for the largest uniform: the branch is unreachable from generated uniforms
    for T in (1.0, 1 - 2.0 ** -52, 1 + 2.0 ** -52, 0.9999995, 1.0000003):
        assert (1 - 2.0 ** -53) * T < T


def test_sampler_refuses_bad_norm():
    psi = np.zeros(4, complex)
    psi[0] = 1.01
    with pytest.raises(oracle.OracleError):
        oracle.sample(psi, oracle.uniforms(1, 10))


# ---------------------------------------------------------------- O9 XEB
def test_xeb_uniform_is_zero_and_ideal_is_fstar():
    text = emit_qasm(generate(3, 4, 12, "ABCDCDAB", seed=2))
    psi = oracle.build_state(text)
    n, S = 12, 200000
    u = oracle.uniforms(99, S)
    xu = np.floor(u * (1 << n)).astype(np.uint64)
    F, sig, _ = oracle.xeb(psi, xu)
    assert abs(F) <= 5 * sig
    x, _ = oracle.sample(psi, oracle.uniforms(100, S))
    F, sig, mp = oracle.xeb(psi, x)
    Fs = oracle.fstar(psi)
    assert abs(F - Fs) <= 5 * sig
    # brute-force definition of F and sigma (V14)
    p = np.abs(psi[x.astype(np.int64)]) ** 2
    assert abs(F - ((1 << n) * p.mean() - 1)) < 1e-12
    assert abs(sig - (1 << n) * p.std(ddof=1) / math.sqrt(S)) < 1e-12
    assert abs(Fs - ((1 << n) * (np.abs(psi) ** 4).sum() - 1)) < 1e-12


def test_porter_thomas_fstar_near_one():
    # deep random circuits: 2^n p ~ Exp(1) => F* ~ 2 * 2^n / (2^n + 1) - 1 ~ 1
    psi = oracle.build_state(config_qasm("c2", n_qubits=16, rows=4, cols=4, cycles=20))
    assert abs(oracle.fstar(psi) - 1) < 0.1


def test_xeb_rejects_out_of_range_bitstring():
    psi = oracle.build_state("OPENQASM 2.0;\nqreg q[2];\n")
    with pytest.raises(oracle.OracleError):
        oracle.xeb(psi, np.array([4], np.uint64))
