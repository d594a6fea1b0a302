"""ctypes wrapper around oracle/rcs_oracle.c (fp64 CPU oracle).

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py cpu_baseline /
--impl reference).  Builds liboracle with gcc + OpenMP on first use.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rcs_oracle.c")
LIB = os.path.join(HERE, "librcs_oracle.so")

KINDS = {0: "sx", 1: "sy", 2: "sw", 3: "rz", 4: "fsim"}
KIND_ID = {v: k for k, v in KINDS.items()}
ERRORS = {1: "PARSE", 2: "UNKNOWN_GATE", 3: "QUBIT_RANGE", 4: "ARITY", 5: "MEMORY",
          6: "NORM", 7: "SIZE", 8: "ARG"}


class OracleError(RuntimeError):
    def __init__(self, code, msg="", line=0, col=0):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        self.line, self.col = line, col
        super().__init__(f"{self.name}: {msg} (line {line}, col {col})")


def build_oracle(force: bool = False) -> str:
    """Compile rcs_oracle.c -> librcs_oracle.so (plain -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off",
                               "-fPIC", "-shared", SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build_oracle())
        u64p = C.POINTER(C.c_uint64)
        dp = C.POINTER(C.c_double)
        lib.orc_parse.argtypes = [C.c_char_p, C.c_long, C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.c_char_p, C.c_int]
        lib.orc_parse.restype = C.c_int
        lib.orc_free.argtypes = [C.c_void_p]
        for f in ("orc_n_qubits", "orc_n_gates", "orc_n_moments", "orc_n_measure"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.c_int
        lib.orc_get_gate.argtypes = [C.c_void_p, C.c_int] + [C.POINTER(C.c_int)] * 3 + [dp, dp, C.POINTER(C.c_int)]
        lib.orc_gate_matrix.argtypes = [C.c_int, C.c_double, C.c_double, dp]
        lib.orc_apply_gate.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double]
        lib.orc_build_state.argtypes = [C.c_void_p, dp, C.c_int]
        lib.orc_build_state.restype = C.c_int
        lib.orc_total_prob.argtypes = [dp, C.c_int]
        lib.orc_total_prob.restype = C.c_double
        lib.orc_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, dp]
        lib.orc_sample.argtypes = [dp, C.c_int, dp, C.c_uint64, u64p, C.c_double, dp]
        lib.orc_sample.restype = C.c_int
        lib.orc_xeb.argtypes = [dp, C.c_int, u64p, C.c_uint64, dp, dp, dp]
        lib.orc_xeb.restype = C.c_int
        lib.orc_fstar.argtypes = [dp, C.c_int]
        lib.orc_fstar.restype = C.c_double
        lib.orc_num_threads.restype = C.c_int
        lib.orc_set_num_threads.argtypes = [C.c_int]
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


@dataclass
class Gate:
    kind: str
    qubits: tuple
    theta: float
    phi: float
    moment: int


class Oracle:
    """A parsed circuit (O1)."""

    def __init__(self, handle):
        self._h = handle
        L = _L()
        self.n_qubits = L.orc_n_qubits(handle)
        self.n_moments = L.orc_n_moments(handle)
        self.n_measure = L.orc_n_measure(handle)
        self.gates = []
        k, q0, q1, m = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        th, ph = C.c_double(), C.c_double()
        for i in range(L.orc_n_gates(handle)):
            L.orc_get_gate(handle, i, C.byref(k), C.byref(q0), C.byref(q1), C.byref(th), C.byref(ph), C.byref(m))
            qs = (q0.value,) if q1.value < 0 else (q0.value, q1.value)
            self.gates.append(Gate(KINDS[k.value], qs, th.value, ph.value, m.value))

    def __del__(self):
        try:
            if self._h:
                _L().orc_free(self._h)
        except Exception:
            pass

    def stats(self):
        cnt = {k: 0 for k in KIND_ID}
        for g in self.gates:
            cnt[g.kind] += 1
        return dict(n_qubits=self.n_qubits, n_moments=self.n_moments, n_gates=len(self.gates), **cnt)

    def build_state(self, max_gates: int = -1) -> np.ndarray:
        psi = np.empty(1 << self.n_qubits, dtype=np.complex128)
        _L().orc_build_state(self._h, _dp(psi.view(np.float64)), max_gates)
        return psi


def parse(text: str) -> Oracle:
    b = text.encode()
    h = C.c_void_p()
    line, col = C.c_int(0), C.c_int(0)
    msg = C.create_string_buffer(256)
    rc = _L().orc_parse(b, len(b), C.byref(h), C.byref(line), C.byref(col), msg, 256)
    if rc:
        raise OracleError(rc, msg.value.decode(), line.value, col.value)
    return Oracle(h.value)


def gate_matrix(kind: str, theta: float = 0.0, phi: float = 0.0) -> np.ndarray:
    d = 4 if kind == "fsim" else 2
    out = np.zeros(d * d, dtype=np.complex128)
    _L().orc_gate_matrix(KIND_ID[kind], theta, phi, _dp(out.view(np.float64)))
    return out.reshape(d, d)


def apply_gate(psi: np.ndarray, kind: str, qubits, theta: float = 0.0, phi: float = 0.0) -> None:
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    n = int(psi.size).bit_length() - 1
    q1 = qubits[1] if len(qubits) > 1 else -1
    _L().orc_apply_gate(_dp(psi.view(np.float64)), n, KIND_ID[kind], qubits[0], q1, theta, phi)


def build_state(text_or_circ, max_gates: int = -1) -> np.ndarray:
    c = parse(text_or_circ) if isinstance(text_or_circ, str) else text_or_circ
    return c.build_state(max_gates)


def total_prob(psi: np.ndarray) -> float:
    n = int(psi.size).bit_length() - 1
    return _L().orc_total_prob(_dp(psi.view(np.float64)), n)


def uniforms(seed: int, count: int, offset: int = 0) -> np.ndarray:
    u = np.empty(count, dtype=np.float64)
    _L().orc_uniforms(seed, offset, count, _dp(u))
    return u


def sample(psi: np.ndarray, u: np.ndarray, norm_tol: float = 1e-6):
    """Returns (x, T)."""
    n = int(psi.size).bit_length() - 1
    u = np.ascontiguousarray(u, dtype=np.float64)
    x = np.empty(u.size, dtype=np.uint64)
    T = C.c_double()
    rc = _L().orc_sample(_dp(psi.view(np.float64)), n, _dp(u), u.size, _u64p(x), norm_tol, C.byref(T))
    if rc:
        raise OracleError(rc, "sample refused")
    return x, T.value


def xeb(psi: np.ndarray, x: np.ndarray):
    """Returns (F, sigma, mean_p)."""
    n = int(psi.size).bit_length() - 1
    x = np.ascontiguousarray(x, dtype=np.uint64)
    F, s, m = C.c_double(), C.c_double(), C.c_double()
    rc = _L().orc_xeb(_dp(psi.view(np.float64)), n, _u64p(x), x.size, C.byref(F), C.byref(s), C.byref(m))
    if rc:
        raise OracleError(rc, "xeb refused")
    return F.value, s.value, m.value


def fstar(psi: np.ndarray) -> float:
    n = int(psi.size).bit_length() - 1
    return _L().orc_fstar(_dp(psi.view(np.float64)), n)


def num_threads() -> int:
    return _L().orc_num_threads()


def set_num_threads(n: int) -> None:
    """Host threads for the oracle's parallel loops (bench.py times the oracle on all host cores)."""
    _L().orc_set_num_threads(int(n))
