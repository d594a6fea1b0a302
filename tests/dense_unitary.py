"""Independent dense 2^n x 2^n checker (NumPy) used to pin the oracle (n <= 10).

Each gate is embedded as an explicit 2^n x 2^n operator built by brute-force index
enumeration (no strided loops, no bit tricks shared with the oracle), the operators are
multiplied in source order, and the product is applied to e_0.  Gate matrices come from
oracle.gate_matrix, which tests/test_oracle_pins.py pins separately by closed-form
properties (sqrt(U)^2 = U, unitarity, fSim closed forms).
"""
import numpy as np


def embed(M: np.ndarray, qubits, n: int) -> np.ndarray:
    """Operator on n qubits acting as M on `qubits` (M's basis index = sum_k b_{qubits[k]} 2^k)."""
    N = 1 << n
    U = np.zeros((N, N), dtype=np.complex128)
    k = len(qubits)
    for col in range(N):
        c = sum(((col >> q) & 1) << j for j, q in enumerate(qubits))
        rest = col
        for q in qubits:
            rest &= ~(1 << q)
        for r in range(1 << k):
            row = rest
            for j, q in enumerate(qubits):
                if (r >> j) & 1:
                    row |= 1 << q
            U[row, col] = M[r, c]
    return U


def kron_1q(M: np.ndarray, q: int, n: int) -> np.ndarray:
    """Second, structurally different embedding for 1q gates: I (x) ... (x) M (x) ... (x) I,
    qubit 0 = rightmost Kronecker factor."""
    return np.kron(np.kron(np.eye(1 << (n - q - 1)), M), np.eye(1 << q))


def circuit_unitary(gates, n: int, gate_matrix) -> np.ndarray:
    U = np.eye(1 << n, dtype=np.complex128)
    for g in gates:
        M = gate_matrix(g.kind, g.theta, g.phi)
        U = embed(M, g.qubits, n) @ U
    return U


def dense_state(gates, n: int, gate_matrix) -> np.ndarray:
    return circuit_unitary(gates, n, gate_matrix)[:, 0].copy()
