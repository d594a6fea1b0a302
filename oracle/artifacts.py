"""Oracle for the paper's stage-2/3 artifacts: snapshot file, shot sharding,
per-job seeds, result-file aggregation.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py): written from the text,
plain Python (struct + hashlib), independent of the library.

  O10 snapshot (SPEC snapshot-store S:181-214, PAPER §3.2 l.37 "written to a shared file
      system"; reading F3-1): header "RCSS" | u32 version 1 | u32 n | u64 16*2^n |
      SHA-256(payload), then (re, im) little-endian float64 in index order.
  O11 shard_shots ("2.5x10^6/N measurement shots"): q = S // N,
      the first S mod N jobs get q + 1.
  O12 job_seed (reading F3-2): SplitMix64 finalizer of base + 0x9E3779B97F4A7C15 (job + 1),
      all arithmetic mod 2^64.
  O13 xeb_from_probs (PAPER l.39 / §5.1; reading V14): F = 2^n mean(p) - 1,
      sigma = 2^n stdev(p, ddof=1) / sqrt(S).
  O14 bitstring text (reading F3-3): format(x, f"0{n}b") -- qubit n-1 first, qubit 0 last.
"""
from __future__ import annotations

import hashlib
import math
import os
import struct

import numpy as np

MAGIC = b"RCSS"
VERSION = 1
HEADER = struct.Struct("<4sIIQ32s")   # 52 bytes
M64 = (1 << 64) - 1


class SnapshotError(RuntimeError):
    pass


def snapshot_bytes(psi) -> bytes:
    """O10: the complete file content for a state vector (complex, any precision -> float64)."""
    a = np.ascontiguousarray(np.asarray(psi, dtype=np.complex128))
    n = int(a.size).bit_length() - 1
    if a.size != 1 << n:
        raise ValueError("state length is not a power of two")
    payload = a.astype("<c16").tobytes()
    return HEADER.pack(MAGIC, VERSION, n, len(payload), hashlib.sha256(payload).digest()) + payload


def save_snapshot(psi, path: str) -> bytes:
    data = snapshot_bytes(psi)
    tmp = f"{path}.tmp.{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)
    return data[20:52]


def read_header(data: bytes) -> dict:
    if len(data) < HEADER.size:
        raise SnapshotError("truncated header")
    magic, ver, n, nbytes, digest = HEADER.unpack_from(data)
    if magic != MAGIC:
        raise SnapshotError("bad magic")
    if ver != VERSION:
        raise SnapshotError("unsupported version")
    if nbytes != 16 << n:
        raise SnapshotError("inconsistent header")
    return {"n_qubits": n, "payload_bytes": nbytes, "digest": digest}


def load_snapshot(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    h = read_header(data)
    payload = data[HEADER.size:HEADER.size + h["payload_bytes"]]
    if len(payload) != h["payload_bytes"]:
        raise SnapshotError("truncated payload")
    if hashlib.sha256(payload).digest() != h["digest"]:
        raise SnapshotError("digest mismatch")
    return np.frombuffer(payload, dtype="<c16").astype(np.complex128)


def shard_shots(total: int, n_jobs: int) -> list:
    """O11."""
    if n_jobs < 1:
        raise ValueError("n_jobs must be >= 1")
    q, r = divmod(total, n_jobs)
    return [q + (1 if j < r else 0) for j in range(n_jobs)]


def job_seed(base_seed: int, job_id: int) -> int:
    """O12."""
    z = (base_seed + 0x9E3779B97F4A7C15 * (job_id + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def xeb_from_probs(n: int, p) -> tuple:
    """O13: (F, sigma, mean_p) over the listed ideal probabilities (one per shot)."""
    p = np.asarray(p, dtype=np.float64)
    S = p.size
    mean = math.fsum(p) / S
    var = math.fsum((p - mean) ** 2) / (S - 1) if S > 1 else 0.0
    return math.ldexp(mean, n) - 1.0, math.ldexp(math.sqrt(var), n) / math.sqrt(S), mean


def bitstring(x: int, n: int) -> str:
    """O14."""
    return format(int(x), f"0{n}b")
