"""Seeded Sycamore-style random-circuit generator -> QASM text.

This module is the ONE piece shared by the oracle side and the CUDA side: it
only produces the input circuit (QASM text).  It contains none of the method's
arithmetic: no gate matrices, no state, no sampling, no XEB.

Paper: PAPER.md §3.1 (lines 29-31) names the workload -- Sycamore random
circuits, "gate pattern EFGH" (14 cycles, fidelity) and "ABCDCDAB" (20 cycles,
performance) -- and §3.2 (line 34) says circuits are "constructed from Google's
QASM-format files".  The paper gives no geometry, gate choice rule or angles,
so this generator follows the readings fixed in DESIGN.md §3 / SURVEY.md §8.0:

* V6  grid rows x cols, qubit = r*cols + c; coupler classes
      A/B = horizontal (r,c)-(r,c+1), c even/odd;
      C/D = vertical   (r,c)-(r+1,c), r even/odd;  E=C, F=D, G=A, H=B.
      Within a class couplers are ordered by (q0, q1) ascending.
* V7  cycle i = one moment of 1q gates on every qubit, then one moment of
      fSim on class letters[i mod len(letters)]; no trailing half cycle
      (SPEC S:54).
* V8  cycle 0: uniform over (sx, sy, sw); later cycles: uniform over the two
      kinds that differ from the qubit's previous kind, in (sx, sy, sw) order
      (SPEC S:54).
* V9  PRNG: SplitMix64 seeded with `seed`; stream order: for every coupler
      (class A, B, C, D; in-class order) one draw for theta jitter then one for
      phi jitter; then per cycle, per qubit ascending, next()%3 (cycle 0) or
      next()%2 (SPEC S:89 asks for a documented counter-based stream).
* V10 fSim angles theta = pi/2 + J*(2u-1), phi = pi/6 + J*(2u-1) with
      u = (next() >> 11) * 2^-53 and J = `jitter` (0.05 for the benchmark
      configs, 0 for closed-form tests).
* V11 n_qubits <= rows*cols: sites with index >= n_qubits are absent
      (truncated row-major); couplers exist only between present sites.

Angles are printed with %.17g so the text round-trips every double exactly.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

ONE_Q_KINDS = ("sx", "sy", "sw")
# QASM spellings emitted for each kind (Cirq/qsim names)
QASM_NAME = {"sx": "x_1_2", "sy": "y_1_2", "sw": "hz_1_2"}


class SplitMix64:
    """Plain SplitMix64 (Steele, Lea, Flood 2014).  Output k (k = 1, 2, ...) is
    mix(seed + k * GOLDEN)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)


def couplers(rows: int, cols: int, n_qubits: int, letter: str) -> list[tuple[int, int]]:
    """Coupler class `letter` on the (truncated) rows x cols grid (V6, V11)."""
    base = {"E": "C", "F": "D", "G": "A", "H": "B"}.get(letter, letter)
    if base not in "ABCD":
        raise ValueError(f"unknown pattern letter {letter!r}")
    out = []
    for r in range(rows):
        for c in range(cols):
            q = r * cols + c
            if q >= n_qubits:
                continue
            if base in "AB":
                if c + 1 < cols and (c % 2 == (0 if base == "A" else 1)):
                    q2 = q + 1
                    if q2 < n_qubits:
                        out.append((q, q2))
            else:
                if r + 1 < rows and (r % 2 == (0 if base == "C" else 1)):
                    q2 = q + cols
                    if q2 < n_qubits:
                        out.append((q, q2))
    out.sort()
    return out


@dataclass
class Gate:
    kind: str                 # "sx" | "sy" | "sw" | "rz" | "fsim"
    qubits: tuple
    params: tuple = ()


@dataclass
class Circuit:
    n_qubits: int
    moments: list = field(default_factory=list)   # list[list[Gate]]

    @property
    def gates(self):
        return [g for m in self.moments for g in m]


def generate(rows: int, cols: int, cycles: int, pattern: str, seed: int,
             n_qubits: int | None = None, jitter: float = 0.05,
             two_qubit: bool = True) -> Circuit:
    """Deterministic Sycamore-style circuit (SPEC S:51-59 + V6-V11).

    two_qubit=False drops every fSim moment (product-state circuit used for
    closed-form full-scale pins)."""
    if not pattern:
        raise ValueError("empty pattern")
    if rows * cols < 1 or cycles < 0:
        raise ValueError("bad grid / cycles")
    n = rows * cols if n_qubits is None else n_qubits
    if not (1 <= n <= rows * cols):
        raise ValueError("n_qubits must be in [1, rows*cols]")
    rng = SplitMix64(seed)
    # per-coupler angle jitter, classes in A, B, C, D order (V9, V10)
    angles = {}
    for cls in "ABCD":
        for cp in couplers(rows, cols, n, cls):
            ut = rng.uniform()
            up = rng.uniform()
            angles[cp] = (math.pi / 2 + jitter * (2 * ut - 1),
                          math.pi / 6 + jitter * (2 * up - 1))
    circ = Circuit(n)
    prev = [None] * n
    for cyc in range(cycles):
        layer = []
        for q in range(n):
            if cyc == 0:
                kind = ONE_Q_KINDS[rng.next() % 3]
            else:
                choices = [k for k in ONE_Q_KINDS if k != prev[q]]
                kind = choices[rng.next() % 2]
            prev[q] = kind
            layer.append(Gate(kind, (q,)))
        circ.moments.append(layer)
        if two_qubit:
            letter = pattern[cyc % len(pattern)]
            layer2 = [Gate("fsim", cp, angles[cp]) for cp in couplers(rows, cols, n, letter)]
            circ.moments.append(layer2)
    return circ


def fmt(x: float) -> str:
    return "%.17g" % x


def emit_qasm(circ: Circuit, measure: bool = False) -> str:
    """Canonical QASM emission; one `barrier` per moment end."""
    n = circ.n_qubits
    lines = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{n}];"]
    if measure:
        lines.append(f"creg c[{n}];")
    for m in circ.moments:
        for g in m:
            if g.kind in QASM_NAME:
                lines.append(f"{QASM_NAME[g.kind]} q[{g.qubits[0]}];")
            elif g.kind == "rz":
                lines.append(f"rz({fmt(g.params[0])}) q[{g.qubits[0]}];")
            elif g.kind == "fsim":
                lines.append(f"fsim({fmt(g.params[0])},{fmt(g.params[1])}) "
                             f"q[{g.qubits[0]}],q[{g.qubits[1]}];")
            else:
                raise ValueError(g.kind)
        lines.append("barrier q;")
    if measure:
        for q in range(n):
            lines.append(f"measure q[{q}] -> c[{q}];")
    return "\n".join(lines) + "\n"


# The benchmark configurations of BASELINE.json, as (rows, cols, n, cycles, pattern, shots)
CONFIGS = {
    "c1": dict(rows=3, cols=4, n_qubits=12, cycles=14, pattern="EFGH", shots=10_000),
    "c2": dict(rows=4, cols=6, n_qubits=24, cycles=20, pattern="ABCDCDAB", shots=100_000),
    "c3": dict(rows=4, cols=8, n_qubits=32, cycles=14, pattern="EFGH", shots=1_000_000),
    "c4": dict(rows=6, cols=6, n_qubits=34, cycles=20, pattern="ABCDCDAB", shots=2_500_000),
    "c5": dict(rows=6, cols=6, n_qubits=36, cycles=20, pattern="ABCDCDAB", shots=2_500_000),
    # weak-scaling extras
    "w33": dict(rows=3, cols=11, n_qubits=33, cycles=20, pattern="ABCDCDAB", shots=2_500_000),
    "w35": dict(rows=5, cols=7, n_qubits=35, cycles=20, pattern="ABCDCDAB", shots=2_500_000),
}
SHOT_SEED = 2512
HEADLINE_SEED = 1


def config_qasm(name: str, seed: int = HEADLINE_SEED, jitter: float = 0.05, **over) -> str:
    cfg = dict(CONFIGS[name])
    cfg.pop("shots")
    cfg.update(over)
    return emit_qasm(generate(cfg["rows"], cfg["cols"], cfg["cycles"], cfg["pattern"], seed,
                              n_qubits=cfg["n_qubits"], jitter=jitter,
                              two_qubit=cfg.get("two_qubit", True)))


def random_qasm(n: int, depth: int, seed: int, rz: bool = True) -> str:
    """Random (non-grid) circuit over all gate kinds for small-n parity tests:
    arbitrary qubit pairs (incl. reversed order), rz gates, random angles."""
    rng = SplitMix64(seed ^ 0xA5A5A5A5)
    lines = ["OPENQASM 2.0;", f"qreg q[{n}];"]
    for _ in range(depth):
        r = rng.next() % (5 if rz else 4)
        if r < 3 or n < 2:
            lines.append(f"{QASM_NAME[ONE_Q_KINDS[r % 3]]} q[{rng.next() % n}];")
        elif r == 3:
            a = rng.next() % n
            b = (a + 1 + rng.next() % (n - 1)) % n
            th = (rng.uniform() * 2 - 1) * math.pi
            ph = (rng.uniform() * 2 - 1) * math.pi
            lines.append(f"fsim({fmt(th)},{fmt(ph)}) q[{a}],q[{b}];")
        else:
            lines.append(f"rz({fmt((rng.uniform() * 2 - 1) * 4)}) q[{rng.next() % n}];")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser(description="emit a Sycamore-style RCS circuit as QASM")
    ap.add_argument("config", nargs="?", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=HEADLINE_SEED)
    ap.add_argument("--jitter", type=float, default=0.05)
    a = ap.parse_args()
    print(config_qasm(a.config, a.seed, a.jitter), end="")
