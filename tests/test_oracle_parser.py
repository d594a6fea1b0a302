"""Oracle parser (O1) and workload generator pins."""
import json
import os
import re

import numpy as np
import pytest

import oracle
from rcs_workload import CONFIGS, config_qasm, couplers, emit_qasm, generate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_fsim_parse_example():
    g = gold("spec_examples.json")["fsim_parse"]
    c = oracle.parse(g["qasm"])
    assert c.n_qubits == g["n_qubits"] and c.n_moments == g["n_moments"]
    assert len(c.gates) == 1 and c.gates[0].kind == "fsim"
    assert c.gates[0].theta == g["theta"] and c.gates[0].phi == g["phi"]


def test_empty_body():
    c = oracle.parse('OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[5];\n')
    assert c.n_qubits == 5 and c.n_moments == 0 and c.gates == []


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_gate_count_equals_text_scan(cfg):
    # gate count equals an independent line scan of the same file
    t = config_qasm(cfg)
    c = oracle.parse(t)
    scan = [ln for ln in t.splitlines() if re.match(r"^(x_1_2|y_1_2|hz_1_2|rz|fsim)\b", ln)]
    assert len(c.gates) == len(scan)
    one = sum(1 for g in c.gates if len(g.qubits) == 1)
    two = len(c.gates) - one
    assert [one, two] == gold("coupler_classes.json")["gate_counts"][cfg]


def test_expressions_and_aliases():
    c = oracle.parse("OPENQASM 2.0;\nqreg q[3];\nsx q[0]; sy q[1]; sw q[2];\n"
                     "rz(-pi/4) q[0];\nfsim(pi/2, 3*pi/6 - 2*pi/6) q[2],q[0];\nrz(1.5e-1) q[1];\n")
    k = [g.kind for g in c.gates]
    assert k == ["sx", "sy", "sw", "rz", "fsim", "rz"]
    assert c.gates[3].phi == -np.pi / 4
    assert abs(c.gates[4].theta - np.pi / 2) < 1e-15 and abs(c.gates[4].phi - np.pi / 6) < 1e-15
    assert c.gates[4].qubits == (2, 0)
    assert c.gates[5].phi == 0.15


def test_moments_barrier_and_clash():
    c = oracle.parse("OPENQASM 2.0;\nqreg q[3];\nsx q[0];\nsx q[1];\nsx q[0];\nbarrier q;\nsy q[2];\n")
    assert [g.moment for g in c.gates] == [0, 0, 1, 2]
    assert c.n_moments == 3


@pytest.mark.parametrize("text,code,line,col", [
    ("OPENQASM 2.0;\nqreg q[2];\nfoo q[0];\n", "UNKNOWN_GATE", 3, 1),
    ("OPENQASM 2.0;\nqreg q[2];\nsx q[2];\n", "QUBIT_RANGE", 3, 6),
    ("OPENQASM 2.0;\nqreg q[2];\nfsim(0.1) q[0],q[1];\n", "ARITY", 3, 1),
    ("OPENQASM 2.0;\nqreg q[2];\nsx q[0],q[1];\n", "ARITY", 3, 1),
    ("OPENQASM 2.0;\nqreg q[2];\nfsim(1,2) q[1],q[1];\n", "ARITY", 3, 1),
    ("OPENQASM 2.0;\nqreg q[2];\n  sx q[0]\n", "PARSE", 4, 1),
    ("OPENQASM 2.0;\nsx q[0];\n", "PARSE", 2, 1),
])
def test_errors_report_line_and_column(text, code, line, col):
    with pytest.raises(oracle.OracleError) as e:
        oracle.parse(text)
    assert e.value.name == code
    assert (e.value.line, e.value.col) == (line, col)


def test_measure_recorded_and_ignored():
    t = emit_qasm(generate(1, 3, 2, "A", 1), measure=True)
    c = oracle.parse(t)
    assert c.n_measure == 3 and len(c.gates) == 3 * 2 + 1 * 2


# ---------------------------------------------------------------- generator
def test_generator_small_structure():
    c = generate(1, 2, 1, "A", 7)
    assert len(c.moments) == 2 and len(c.moments[0]) == 2 and len(c.moments[1]) <= 1


def test_generator_determinism_and_roundtrip():
    a, b = config_qasm("c2"), config_qasm("c2")
    assert a == b
    c = oracle.parse(a)
    # emit -> parse -> same gates, angles bit-exact (%.17g)
    circ = generate(**{k: v for k, v in CONFIGS["c2"].items() if k in ("rows", "cols", "cycles", "pattern")},
                    seed=1, n_qubits=24)
    src = [g for m in circ.moments for g in m]
    assert len(src) == len(c.gates)
    for s, g in zip(src, c.gates):
        assert s.kind == g.kind and tuple(s.qubits) == g.qubits
        if s.kind == "fsim":
            assert (s.params[0], s.params[1]) == (g.theta, g.phi)


def test_generator_no_repeat_rule_and_histogram():
    from scipy.stats import chi2
    circ = generate(4, 4, 14, "EFGH", 1)
    prev = {}
    hist = {"sx": 0, "sy": 0, "sw": 0}
    for m in circ.moments:
        for g in m:
            if len(g.qubits) == 1:
                q = g.qubits[0]
                assert prev.get(q) != g.kind
                prev[q] = g.kind
                hist[g.kind] += 1
    tot = sum(hist.values())
    stat = sum((v - tot / 3) ** 2 / (tot / 3) for v in hist.values())
    assert stat < chi2.ppf(0.99, 2)


def test_coupler_classes_golden():
    for case in gold("coupler_classes.json")["cases"]:
        got = [len(couplers(case["rows"], case["cols"], case["n"], L)) for L in "ABCD"]
        assert got == case["ABCD"]
    # E=C, F=D, G=A, H=B (reading V6)
    for a, b in zip("EFGH", "CDAB"):
        assert couplers(4, 6, 24, a) == couplers(4, 6, 24, b)
    # couplers of one class are disjoint (moment exclusivity)
    for L in "ABCD":
        qs = [q for cp in couplers(6, 6, 34, L) for q in cp]
        assert len(qs) == len(set(qs))
