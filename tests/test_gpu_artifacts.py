"""GPU tests of paper stages 2-4: snapshot save/load through the C ABI against
the oracle's file format, independent sampler jobs and the aggregated XEB."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import artifacts as A
from rcs_workload import SHOT_SEED, config_qasm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rcs(cuda_ok):
    from paper_2512_07311_b200 import build
    build.build()
    import paper_2512_07311_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(rcs):
    return rcs.Context(0)


def test_snapshot_bytes_equal_oracle_format(rcs, ctx, tmp_path):
    """The library's file == the oracle's file for the same (complex64 -> float64) amplitudes."""
    st = rcs.State.build(ctx, rcs.Circuit.from_qasm(config_qasm("c1")))
    p = str(tmp_path / "g.rcss")
    dg = st.save_snapshot(p)
    psi = st.copy_out()
    assert open(p, "rb").read() == A.snapshot_bytes(psi.astype(np.complex128))
    assert dg == A.read_header(open(p, "rb").read(52))["digest"]
    assert not [f for f in os.listdir(tmp_path) if ".tmp." in f]       # atomic write left no temp file


def test_snapshot_roundtrip_sampling_and_errors(rcs, ctx, tmp_path):
    st = rcs.State.build(ctx, rcs.Circuit.from_qasm(config_qasm("c2")))
    p = str(tmp_path / "c2.rcss")
    st.save_snapshot(p)
    before = open(p, "rb").read()
    ld = rcs.State.load_snapshot(ctx, p)
    assert np.array_equal(ld.copy_out().view(np.uint64), st.copy_out().view(np.uint64))   # bit-identical
    assert open(p, "rb").read() == before                                                   # read-only
    assert np.array_equal(ld.sample(50_000, seed=SHOT_SEED), st.sample(50_000, seed=SHOT_SEED))
    assert abs(ld.xeb(st.sample(1000, seed=3))["F"] - st.xeb(st.sample(1000, seed=3))["F"]) == 0
    raw = bytearray(before)
    raw[52 + 8 * 12345] ^= 0x10
    q = str(tmp_path / "bad.rcss")
    open(q, "wb").write(raw)
    with pytest.raises(rcs.RcsError) as e:
        rcs.State.load_snapshot(ctx, q)
    assert e.value.status == "RCS_ERR_DIGEST"
    open(q, "wb").write(before[:-16])
    with pytest.raises(rcs.RcsError) as e:
        rcs.State.load_snapshot(ctx, q)
    assert e.value.status == "RCS_ERR_FORMAT"


def test_load_oracle_fp64_snapshot(rcs, ctx, tmp_path):
    """An fp64 state written by the oracle loads as its round-to-nearest complex64 and samples
    like the oracle (G17 excuse band)."""
    text = config_qasm("c1")
    ref = oracle.build_state(text)
    p = str(tmp_path / "o.rcss")
    A.save_snapshot(ref, p)
    ld = rcs.State.load_snapshot(ctx, p)
    assert np.array_equal(ld.copy_out(), ref.astype(np.complex64))
    u = oracle.uniforms(SHOT_SEED, 10_000)
    x_o, _ = oracle.sample(ref, u)
    x_g = ld.sample(10_000, seed=SHOT_SEED)
    C = np.cumsum(np.abs(ref) ** 2)
    d = np.nonzero(x_g != x_o)[0]
    xg = x_g[d].astype(np.int64)
    t = u[d] * C[-1]
    lo = np.where(xg > 0, C[np.maximum(xg - 1, 0)], 0.0) - 1e-6
    assert ((t >= lo) & (t <= C[xg] + 1e-6)).all()


def test_worker_result_files(rcs, ctx, tmp_path):
    """distinct jobs -> distinct seeds; sum(counts) = shots; p_ideal = |psi_x|^2;
    rerun identical except timings; an existing result file is never overwritten."""
    from paper_2512_07311_b200 import jobs
    text = config_qasm("c1")
    ref = oracle.build_state(text)
    st = rcs.State.build(ctx, rcs.Circuit.from_qasm(text))
    snap = str(tmp_path / "s.rcss")
    st.save_snapshot(snap)
    d1, d2 = tmp_path / "a", tmp_path / "b"
    d1.mkdir()
    d2.mkdir()
    h1 = jobs.run_worker(snap, 2500, 2512, 1, str(d1))
    h2 = jobs.run_worker(snap, 2500, 2512, 2, str(d1))
    assert h1["seed"] == A.job_seed(2512, 1) and h2["seed"] == A.job_seed(2512, 2) and h1["seed"] != h2["seed"]
    head, x, c, p = jobs.read_result(str(d1 / "result_1.jsonl"))
    assert c.sum() == 2500 and head["shots"] == 2500 and head["n_qubits"] == 12
    assert head["timings"]["sample_s"] > 0 and head["timings"]["load_s"] > 0
    a = np.abs(ref[x.astype(np.int64)])
    assert (np.abs(p - a ** 2) <= (2 * a + 1e-5) * 1e-5).all()      # amplitude tolerance 1e-5 (G16)
    np.testing.assert_allclose(p, np.abs(st.copy_out()[x.astype(np.int64)].astype(np.complex128)) ** 2, rtol=1e-6)
    lines = open(d1 / "result_1.jsonl").read().splitlines()
    assert json.loads(lines[1])["bitstring"] == A.bitstring(int(x[0]), 12)
    # the job's draws are the library's sampler with the job seed
    xs = st.sample(2500, seed=h1["seed"])
    ux, uc = np.unique(xs, return_counts=True)
    assert np.array_equal(ux, x) and np.array_equal(uc, c)
    jobs.run_worker(snap, 2500, 2512, 1, str(d2))
    strip = lambda s: [ln for ln in s.splitlines()[1:]]
    assert strip(open(d2 / "result_1.jsonl").read()) == strip(open(d1 / "result_1.jsonl").read())
    with pytest.raises(FileExistsError):
        jobs.run_worker(snap, 2500, 2512, 1, str(d1))


def test_pipeline_fanout_xeb(rcs, tmp_path):
    """Stages 1-4 with 4 independent worker processes: shots shard as PAPER l.38, aggregated XEB
    equals the oracle's XEB of the same bitstrings and is within 5 sigma of F*."""
    from paper_2512_07311_b200 import jobs
    text = config_qasm("c1")
    out = jobs.run_pipeline(text, 10_000, 4, 2512, str(tmp_path / "w"), parallel=2)
    assert out["shots"] == 10_000 and out["jobs"] == 4
    ref = oracle.build_state(text)
    xs = []
    for j in range(4):
        h, x, c, _ = jobs.read_result(str(tmp_path / "w" / f"result_{j}.jsonl"))
        assert h["shots"] == A.shard_shots(10_000, 4)[j]
        xs.append(np.repeat(x, c))
    F_o, s_o, _ = oracle.xeb(ref, np.concatenate(xs))
    assert abs(out["F"] - F_o) <= 1e-3
    assert abs(out["F"] - oracle.fstar(ref)) <= 5 * out["sigma"]
