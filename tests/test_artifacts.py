"""Paper stages 2-4 artifacts without a GPU: the oracle (oracle/artifacts.py)
pinned to SPEC/PAPER values and FIPS test vectors, and the library's host-side functions
(rcs_sha256, rcs_snapshot_info, rcs_shard_shots, rcs_job_seed, rcs_xeb_from_probs) against it."""
import hashlib
import os
import struct

import numpy as np
import pytest

from oracle import artifacts as A


@pytest.fixture(scope="module")
def rcs():
    from paper_2512_07311_b200 import build
    build.build()
    import paper_2512_07311_b200 as m
    return m


# ------------------------------------------------------------------ oracle pins
def test_snapshot_n1_ground_state_bytes():
    """n=1 |0> -> payload 1.0, 0.0, 0.0, 0.0 as little-endian float64."""
    data = A.snapshot_bytes(np.array([1, 0], complex))
    assert data[:4] == b"RCSS" and len(data) == 52 + 32
    assert struct.unpack("<II", data[4:12]) == (1, 1) and struct.unpack("<Q", data[12:20]) == (32,)
    assert data[52:] == struct.pack("<4d", 1.0, 0.0, 0.0, 0.0)
    assert data[20:52] == hashlib.sha256(data[52:]).digest()


def test_snapshot_payload_size_n20():
    """n=20 -> payload_bytes = 16,777,216."""
    hdr = A.read_header(A.snapshot_bytes(np.zeros(1 << 20, complex))[:52])
    assert hdr["payload_bytes"] == 16_777_216 and hdr["n_qubits"] == 20


def test_snapshot_roundtrip_and_corruption(tmp_path):
    """bit-identical round trip; every single-byte payload
    mutation (random offsets) is detected; a bad magic is rejected."""
    rng = np.random.default_rng(1)
    for n in (1, 3, 8):
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        p = str(tmp_path / f"s{n}.rcss")
        A.save_snapshot(psi, p)
        assert np.array_equal(A.load_snapshot(p).view(np.uint64), psi.astype(np.complex128).view(np.uint64))
    raw = bytearray(open(p, "rb").read())
    for off in rng.integers(52, len(raw), 20):
        bad = bytearray(raw)
        bad[off] ^= 1 << int(rng.integers(0, 8))
        open(p, "wb").write(bad)
        with pytest.raises(A.SnapshotError, match="digest"):
            A.load_snapshot(p)
    bad = bytearray(raw)
    bad[0:4] = b"RCSX"
    with pytest.raises(A.SnapshotError, match="magic"):
        A.read_header(bytes(bad))


def test_shard_shots_paper_values():
    """PAPER §5.3: 25,000 shots per job with 100 jobs; Table 2: 2,500 with 1000; SPEC: (10,3)."""
    assert A.shard_shots(2_500_000, 100) == [25_000] * 100
    assert A.shard_shots(2_500_000, 1000) == [2_500] * 1000
    assert A.shard_shots(10, 3) == [4, 3, 3]
    rng = np.random.default_rng(2)
    for _ in range(50):
        s, n = int(rng.integers(0, 10**7)), int(rng.integers(1, 500))
        sh = A.shard_shots(s, n)
        assert sum(sh) == s and max(sh) - min(sh) <= 1


def test_job_seed_is_splitmix64_output():
    """Reading F3-2: job_seed(base, j) is the (j+1)-th SplitMix64 output of the stream seeded
    with `base` -- pinned to the published SplitMix64 vector (tests/golden/splitmix64.json)."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64.json")))
    seed, outs = g["seed"], [int(h, 16) for h in g["outputs_hex"]]
    for j, v in enumerate(outs):
        assert A.job_seed(seed, j) == v
    assert len({A.job_seed(2512, j) for j in range(1000)}) == 1000


def test_xeb_from_probs_closed_forms():
    """V14: uniform p = 2^-n -> F = 0, sigma = 0; p = 2^-(n-1) -> F = 1."""
    F, s, m = A.xeb_from_probs(10, [2.0 ** -10] * 100)
    assert F == 0 and s == 0
    F, s, m = A.xeb_from_probs(10, [2.0 ** -9] * 7)
    assert F == 1


# ------------------------------------------------------------------ library host functions vs oracle
def test_library_sha256_fips_vectors_and_random(rcs):
    assert rcs.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert rcs.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert rcs.sha256(b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq").hex() == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"
    rng = np.random.default_rng(3)
    for n in (1, 55, 56, 63, 64, 65, 127, 1000, 100_003):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert rcs.sha256(b) == hashlib.sha256(b).digest()


def test_library_snapshot_info_reads_oracle_files(rcs, tmp_path):
    psi = np.exp(1j * np.arange(64))
    p = str(tmp_path / "a.rcss")
    dg = A.save_snapshot(psi, p)
    info = rcs.snapshot_info(p)
    assert info == {"n_qubits": 6, "payload_bytes": 1024, "digest": dg}
    raw = bytearray(open(p, "rb").read())
    for off, val, status in ((0, b"X", "RCS_ERR_FORMAT"), (4, b"\x02", "RCS_ERR_FORMAT"), (12, b"\x01", "RCS_ERR_FORMAT")):
        bad = bytearray(raw)
        bad[off:off + 1] = val
        q = str(tmp_path / "bad.rcss")
        open(q, "wb").write(bad)
        with pytest.raises(rcs.RcsError) as e:
            rcs.snapshot_info(q)
        assert e.value.status == status
    with pytest.raises(rcs.RcsError) as e:
        rcs.snapshot_info(str(tmp_path / "missing.rcss"))
    assert e.value.status == "RCS_ERR_IO"


def test_library_shard_seed_xeb_match_oracle(rcs):
    for s, n in ((2_500_000, 100), (2_500_000, 1000), (10, 3), (7, 9), (0, 4)):
        assert rcs.shard_shots(s, n) == A.shard_shots(s, n)
    with pytest.raises(rcs.RcsError):
        rcs.shard_shots(10, 0)
    for b in (0, 1, 2512, (1 << 64) - 1):
        for j in (0, 1, 99, 12345):
            assert rcs.job_seed(b, j) == A.job_seed(b, j)
    rng = np.random.default_rng(4)
    p = rng.exponential(2.0 ** -20, 100_000)
    r = rcs.xeb_from_probs(20, p)
    F, s, m = A.xeb_from_probs(20, p)
    assert abs(r["F"] - F) <= 1e-12 and abs(r["sigma"] - s) <= 1e-12 * max(1, s) and r["shots"] == p.size
