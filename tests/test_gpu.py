"""GPU parity tests: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star):
  amplitudes  max |d psi| <= 1e-5 and ||d psi||_2 <= 1e-5 (reading G16), norm within 1e-5
  bitstrings  identical except where the uniform lies within 1e-6 of the CDF boundary that
              separates the two picks (reading G17)
  XEB         same-sample |F(x; p_gpu) - F(x; p_oracle)| <= 1e-3 (reading G18)
"""
import math

import numpy as np
import pytest

import oracle
from rcs_workload import SHOT_SEED, config_qasm, emit_qasm, generate, random_qasm

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


def gpu_state(rcs, ctx, text, **kw):
    c = rcs.Circuit.from_qasm(text)
    st = rcs.State.build(ctx, c, **kw)
    return st, st.copy_out().astype(np.complex128)


def check_amps(psi, ref):
    d = psi - ref
    assert np.abs(d).max() <= 1e-5
    assert np.linalg.norm(d) <= 1e-5
    assert abs(np.vdot(psi, psi).real - 1) <= 1e-5


def excused(x_g, x_o, u, p_o):
    """G17: a GPU pick differing from the oracle's is excused iff the oracle CDF interval
    of the GPU pick, widened by 1e-6, contains t = u T_o."""
    C = np.cumsum(p_o)
    T = C[-1]
    t = u * T
    diff = np.nonzero(x_g != x_o)[0]
    xg = x_g[diff].astype(np.int64)
    lo = np.where(xg > 0, C[np.maximum(xg - 1, 0)], 0.0) - 1e-6
    hi = C[xg] + 1e-6
    ok = (t[diff] >= lo) & (t[diff] <= hi)
    return len(diff), int((~ok).sum())


# ------------------------------------------------------------------ state parity
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("seed", range(6))
def test_random_circuits_all_k(rcs, ctx, k, seed):
    n = [1, 2, 5, 7, 10, 13][seed] if k < 6 else [12, 13, 14, 15, 17, 19][seed]
    text = random_qasm(n, 12 * n + 5, 77 + seed)
    ref = oracle.build_state(text)
    st, psi = gpu_state(rcs, ctx, text, fuse_k=k)
    check_amps(psi, ref)
    assert abs(st.norm - 1) <= 1e-5


@pytest.mark.parametrize("k", [4, 6])
@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_baseline_configs_state(rcs, ctx, cfg, k):
    text = config_qasm(cfg)
    ref = oracle.build_state(text)
    st, psi = gpu_state(rcs, ctx, text, fuse_k=k, timing=True)
    check_amps(psi, ref)
    assert st.report["n_passes"] == len(st.pass_times())
    if k == 6:
        assert st.report["n_tc_passes"] > 0


@pytest.mark.parametrize("g", [1, 2, 3])
def test_virtual_global_bitwise_equals_single(rcs, ctx, g):
    text = emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=g))
    ref = oracle.build_state(text)
    _, psi1 = gpu_state(rcs, ctx, text)
    stg, psig = gpu_state(rcs, ctx, text, virtual_global=g)
    assert stg.report["n_remaps"] > 0
    assert np.array_equal(psi1, psig)            # P-invariance of the fused arithmetic
    check_amps(psig, ref)


@pytest.mark.parametrize("n", [21, 26, 29])
def test_transposed_pass_matches_k9(rcs, ctx, n):
    """K12 (blocks without qubits 0..6) against K9 on the same plan: equal up to the tensor
    core's summation order; n = 21 also against the oracle."""
    text = config_qasm("c3", n_qubits=n)
    c = rcs.Circuit.from_qasm(text)
    a = rcs.State.build(ctx, c, fuse_k=6)
    pa = a.copy_out(0, 1 << min(n, 24)).astype(np.complex128)
    na = a.norm
    del a
    b = rcs.State.build(ctx, c, fuse_k=6, tc_kernel="k9")
    pb = b.copy_out(0, 1 << min(n, 24)).astype(np.complex128)
    assert np.abs(pa - pb).max() <= 1e-8 and abs(na - b.norm) <= 1e-7
    if n == 21:
        check_amps(pa, oracle.build_state(text))


@pytest.mark.parametrize("grid", [(4, 5, 12, "ABCDCDAB"), (3, 7, 12, "EFGH"), (4, 6, 15, "ABCDCDAB")])
def test_multi_low_target_blocks_on_k12(rcs, ctx, grid):
    """Blocks with 2-4 targets in positions 0..3 (row 0 of the grid) run on K12 with a lane
    permutation of up to four t bits (round 2; K9 before): equal to the K9 build up to the cross
    terms' rounding order and to the oracle within the BASELINE tolerance."""
    rows, cols, cyc, pat = grid
    text = emit_qasm(generate(rows, cols, cyc, pat, seed=1))
    c = rcs.Circuit.from_qasm(text)
    plan = rcs.Plan(c, 6, 0)
    multi = [it for it in plan.items()[plan.prefix:]
             if it["type"] == "pass" and sum(x < 4 for x in it["pos"]) >= 2]
    assert len(multi) >= 3   # >= 2 low targets: K12 (kPermMulti) for 2, K9 for 3-4
    a = rcs.State.build(ctx, c, fuse_k=6)
    pa = a.copy_out().astype(np.complex128)
    b = rcs.State.build(ctx, c, fuse_k=6, tc_kernel="k9")
    pb = b.copy_out().astype(np.complex128)
    assert np.abs(pa - pb).max() <= 1e-8 and abs(a.norm - b.norm) <= 1e-7
    check_amps(pa, oracle.build_state(text))


@pytest.mark.parametrize("grid", [(3, 7, 12, "ABCDCDAB", 1), (3, 7, 12, "ABCDCDAB", 2)])
def test_row_variant_blocks(rcs, ctx, grid):
    """Blocks on positions 0..5 (grid row 0) run on K12's row variant -- tensor-map TMA load with
    the 128-B swizzle, TMA stores from a 64-B-swizzled staging buffer: equal to the K9 build of
    the same blocks (tc_kernel="norow") up to the cross terms' rounding order, and to the oracle."""
    rows, cols, cyc, pat, seed = grid
    text = emit_qasm(generate(rows, cols, cyc, pat, seed=seed))
    c = rcs.Circuit.from_qasm(text)
    plan = rcs.Plan(c, 6, 0)
    assert any(it["type"] == "pass" and it["pos"] == [0, 1, 2, 3, 4, 5] for it in plan.items()[plan.prefix:])
    a = rcs.State.build(ctx, c, fuse_k=6)
    pa = a.copy_out().astype(np.complex128)
    b = rcs.State.build(ctx, c, fuse_k=6, tc_kernel="norow")
    pb = b.copy_out().astype(np.complex128)
    assert np.abs(pa - pb).max() <= 1e-8 and abs(a.norm - b.norm) <= 1e-7
    check_amps(pa, oracle.build_state(text))


@pytest.mark.parametrize("case", ["c1", "c3_24", "w33_24", "grid20_k4", "idle22"])
def test_product_prefix_matches_passes(rcs, ctx, case):
    """The leading fused blocks on disjoint qubits act on |0...0>: the product-state kernel writes
    their state in one write-only sweep (fp64 block products rounded to complex64, one fixed-order
    complex product) instead of init + passes; both agree with the oracle and with each other
    within the pass rounding.  idle22: qubits 19..21 carry no gate, so the prefix kernel's zero
    path (amplitudes with a |1> outside the prefix) is exercised, rows and single amplitudes."""
    idle = random_qasm(19, 260, 7).replace("qreg q[19];", "qreg q[22];")
    text, k = {"c1": (config_qasm("c1"), 6), "c3_24": (config_qasm("c3", n_qubits=24, rows=4, cols=6), 6),
               "w33_24": (config_qasm("w33", n_qubits=24), 6),
               "grid20_k4": (emit_qasm(generate(4, 5, 12, "ABCDCDAB", seed=2)), 4),
               "idle22": (idle, 6)}[case]
    c = rcs.Circuit.from_qasm(text)
    a = rcs.State.build(ctx, c, fuse_k=k, timing=True)
    pa = a.copy_out().astype(np.complex128)
    b = rcs.State.build(ctx, c, fuse_k=k, product_prefix=False)
    pb = b.copy_out().astype(np.complex128)
    assert a.report["n_prefix"] > 0 and b.report["n_prefix"] == 0
    assert a.report["n_passes"] + a.report["n_prefix"] == b.report["n_passes"]
    assert a.report["n_passes"] == len(a.pass_times()) and a.report["prefix_ms"] > 0
    ref = oracle.build_state(text)
    check_amps(pa, ref)
    check_amps(pb, ref)
    assert np.abs(pa - pb).max() <= 1e-6


@pytest.mark.parametrize("case", ["c2", "c3"])
def test_dynamic_tile_schedule_bitwise(rcs, ctx, case):
    """K12's optional dynamic scheduler hands tiles to the SMs through a device counter; the
    arithmetic of a tile does not depend on the SM that runs it, so the state equals the static
    round-robin schedule (the default) bit for bit (C3: n = 32, the first and last 4M amplitudes)."""
    c = rcs.Circuit.from_qasm(config_qasm(case))
    a = rcs.State.build(ctx, c, fuse_k=6, tc_schedule="dynamic")
    if case == "c3":
        pa = (a.copy_out(0, 1 << 22), a.copy_out((1 << 32) - (1 << 22), 1 << 22))
    else:
        pa = (a.copy_out(),)
    na = a.norm
    a.free()
    b = rcs.State.build(ctx, c, fuse_k=6, tc_schedule="static")
    pb = (b.copy_out(0, 1 << 22), b.copy_out((1 << 32) - (1 << 22), 1 << 22)) if case == "c3" else (b.copy_out(),)
    assert all(np.array_equal(x, y) for x, y in zip(pa, pb))
    assert na == b.norm


@pytest.mark.parametrize("case", ["c2", "c3", "loop"])
def test_tensor_map_runs_bitwise(rcs, ctx, case):
    """K12 fetches tiles whose contiguous runs are short (2^r <= 256 amplitudes) with a few 5-D
    tensor-map TMA requests instead of one bulk copy per run; only the copy engine's request shape
    changes, so the state equals the bulk-copy build bit for bit (C3: n = 32, every pass kind;
    loop: n = 20 with 2 virtual global qubits, pipelined remap chunks as fixed index bits)."""
    if case == "loop":
        c = rcs.Circuit.from_qasm(emit_qasm(generate(4, 5, 10, "ABCDCDAB", seed=3)))
        kw = {"virtual_global": 2, "remap_mode": "loopback"}
    else:
        c = rcs.Circuit.from_qasm(config_qasm(case))
        kw = {}
    def run(tma):
        st = rcs.State.build(ctx, c, fuse_k=6, tc_tma=tma, **kw)
        if case == "c3":
            out = (st.copy_out(0, 1 << 22), st.copy_out((1 << 31) + (5 << 22), 1 << 22),
                   st.copy_out((1 << 32) - (1 << 22), 1 << 22))
        else:
            out = (st.copy_out(),)
        nrm = st.norm
        st.free()
        return out, nrm
    pa, na = run("auto")
    pb, nb = run("bulk")
    assert all(np.array_equal(x, y) for x, y in zip(pa, pb)) and na == nb
    if case != "c3":
        check_amps(pa[0].astype(np.complex128), oracle.build_state(c_text(case)))


def c_text(case):
    return emit_qasm(generate(4, 5, 10, "ABCDCDAB", seed=3)) if case == "loop" else config_qasm(case)


@pytest.mark.parametrize("g", [1, 2, 3])
def test_keep_layout_matches_canonical(rcs, ctx, g):
    """keep_layout skips the final restore; the logical-order CDF over the permuted layout gives
    the same T, shots, probabilities and XEB bit for bit (same block sums, same scan order), and
    canonicalize() then yields the canonical amplitudes."""
    text = emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=10 + g))
    c = rcs.Circuit.from_qasm(text)
    can = rcs.State.build(ctx, c, virtual_global=g)
    kept = rcs.State.build(ctx, c, virtual_global=g, keep_layout=True)
    assert kept.report["layout_kept"] == 1
    assert kept.report["n_remaps"] + kept.report["n_swaps"] < can.report["n_remaps"] + can.report["n_swaps"]
    assert kept.norm == can.norm
    xa = can.sample(200_000, seed=SHOT_SEED)
    xb = kept.sample(200_000, seed=SHOT_SEED)
    assert np.array_equal(xa, xb)
    u = oracle.uniforms(4, 3000)
    u[:3] = [0.0, 1.0 - 2.0 ** -53, 0.5]
    assert np.array_equal(can.sample_uniforms(u), kept.sample_uniforms(u))
    assert np.array_equal(can.probabilities(xa[:5000]), kept.probabilities(xa[:5000]))
    ra, rb = can.xeb(xa), kept.xeb(xa)
    assert (ra["F"], ra["sigma"], ra["mean_p"]) == (rb["F"], rb["sigma"], rb["mean_p"])
    assert abs(ra["fstar"] - rb["fstar"]) <= 1e-12     # sum p^2 accumulated in physical order
    with pytest.raises(rcs.RcsError) as e:
        kept.copy_out()
    assert e.value.status == "RCS_ERR_ARG"
    kept.canonicalize()
    assert np.array_equal(kept.copy_out(), can.copy_out())
    assert np.array_equal(kept.sample(10_000, seed=1), can.sample(10_000, seed=1))


def test_empty_and_tiny_circuits(rcs, ctx):
    for n in (1, 2, 3, 7):
        st, psi = gpu_state(rcs, ctx, f"OPENQASM 2.0;\nqreg q[{n}];\n")
        e = np.zeros(1 << n); e[0] = 1
        assert np.array_equal(psi, e)
        x = st.sample(1000)
        assert (x == 0).all()
    st, psi = gpu_state(rcs, ctx, "OPENQASM 2.0;\nqreg q[1];\nx_1_2 q[0];\n")
    np.testing.assert_allclose(psi, [0.5 + 0.5j, 0.5 - 0.5j], atol=1e-7)


def test_product_state_closed_form_n26(rcs, ctx):
    circ = generate(2, 13, 8, "ABCD", seed=4, two_qubit=False)
    c = oracle.parse(emit_qasm(circ))
    v = [np.array([1, 0], complex) for _ in range(26)]
    for g in c.gates:
        v[g.qubits[0]] = oracle.gate_matrix(g.kind) @ v[g.qubits[0]]
    st = rcs.State.build(ctx, rcs.Circuit.from_qasm(emit_qasm(circ)))
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 1 << 26, 4096)
    full = st.copy_out()
    for x in idx[:4096]:
        a = np.prod([v[q][(x >> q) & 1] for q in range(26)])
        assert abs(full[x] - a) <= 1e-6


# ------------------------------------------------------------------ sampling + XEB parity
@pytest.mark.parametrize("cfg,shots", [("c1", 10_000), ("c2", 100_000)])
def test_sampling_and_xeb_parity(rcs, ctx, cfg, shots):
    text = config_qasm(cfg)
    ref = oracle.build_state(text)
    st, psi = gpu_state(rcs, ctx, text)
    x_g = st.sample(shots, seed=SHOT_SEED)
    u = oracle.uniforms(SHOT_SEED, shots)
    x_o, T_o = oracle.sample(ref, u)
    p_o = np.abs(ref) ** 2
    nd, bad = excused(x_g, x_o, u, p_o)
    assert bad == 0, f"{bad} unexcused of {nd} differing shots"
    # mismatch fraction f ~ 0.75 eps 2^(n/2) for state error eps = ||dpsi||_2
    eps = np.linalg.norm(psi - ref)
    n = int(len(ref)).bit_length() - 1
    assert nd <= max(10, 4 * 0.75 * eps * 2 ** (n / 2) * shots), (nd, eps)
    # XEB: same-sample check and independent comparison
    xr = st.xeb(x_g)
    F_o_same, _, _ = oracle.xeb(ref, x_g)
    assert abs(xr["F"] - F_o_same) <= 1e-3
    F_o, sig_o, _ = oracle.xeb(ref, x_o)
    assert abs(xr["F"] - F_o) <= 1e-3
    assert abs(xr["fstar"] - oracle.fstar(ref)) <= 1e-4
    assert abs(xr["F"] - xr["fstar"]) <= 5 * xr["sigma"]


def dyadic_state(n, K, seed, zero_blocks=(), b=6):
    """K = 4^m non-zero amplitudes of magnitude 2^-m with phases in {1, i, -1, -i}: every
    probability (1/K), block sum and CDF value is exact in fp32, fp64 and any summation order.
    The listed 2^b-amplitude blocks and the last block are all zero (trailing zeros)."""
    rng = np.random.default_rng(seed)
    N = 1 << n
    allowed = np.ones(N, bool)
    for z in list(zero_blocks) + [N // (1 << b) - 1]:
        allowed[z << b:(z + 1) << b] = False
    pos = np.sort(rng.choice(np.nonzero(allowed)[0], K, replace=False))
    psi = np.zeros(N, complex)
    psi[pos] = np.array([1, 1j, -1, -1j])[rng.integers(0, 4, K)] / math.sqrt(K)
    return psi


@pytest.mark.parametrize("case", ["ties8", "n10", "n12_b3"])
def test_sampling_edge_uniforms_vs_oracle(rcs, ctx, case, tmp_path):
    """V13 edge cases on the GPU path, bit-exact against the oracle on states whose CDF is exact:
    u = 0, u = 1 - 2^-53 (largest generated uniform), u = 1 (t = T: the 'last x with p > 0'
    fallback, through the uniform hook), t exactly on CDF boundaries (ties: the next x with
    p > 0), exact zero probabilities, all-zero blocks and a zero tail.  The
    state enters through the snapshot loader (any state, rounded to complex64 exactly)."""
    from oracle.artifacts import save_snapshot
    if case == "ties8":
        psi = np.zeros(8, complex)
        psi[0], psi[2], psi[3] = 0.5, 0.5, 0.5 + 0.5j
        b, K = 6, 4
    elif case == "n10":
        psi, b, K = dyadic_state(10, 256, 1, zero_blocks=(0, 3, 7)), 6, 256
    else:
        psi, b, K = dyadic_state(12, 1024, 2, zero_blocks=(5, 6, 100), b=3), 3, 1024
    path = str(tmp_path / "s.rcss")
    save_snapshot(psi, path)
    st = rcs.State.load_snapshot(ctx, path, block_bits=b)
    assert st.norm == 1.0
    C = np.cumsum(np.abs(psi) ** 2)
    bounds = np.unique(C[(C > 0) & (C < 1)])              # exact CDF values -> t on a boundary
    u = np.concatenate([[0.0, 1 - 2.0 ** -53, 1.0, 0.5], bounds, bounds - 2.0 ** -40,
                        oracle.uniforms(7, 20000)])
    xg = st.sample_uniforms(u)
    xo, T = oracle.sample(psi, u)
    assert T == 1.0
    np.testing.assert_array_equal(xg, xo)
    p = np.abs(psi) ** 2
    assert (p[xg.astype(np.int64)] > 0).all()               # never a zero-probability pick
    last = np.nonzero(p)[0][-1]
    assert xg[1] == last and xg[2] == last                  # u = 1 - 2^-53 and the u = 1 fallback
    st.free()


def test_sample_uniforms_hook_and_offsets(rcs, ctx):
    text = config_qasm("c1")
    ref = oracle.build_state(text)
    st, _ = gpu_state(rcs, ctx, text, block_bits=3)
    u = oracle.uniforms(9, 5000)
    xa = st.sample_uniforms(u)
    xb = st.sample(5000, seed=9)
    assert np.array_equal(xa, xb)
    xc = st.sample(1000, seed=9, offset=2000)
    assert np.array_equal(xc, xb[2000:3000])
    x_o, _ = oracle.sample(ref, u)
    nd, bad = excused(xa, x_o, u, np.abs(ref) ** 2)
    assert bad == 0
    # device output
    xd = st.sample(5000, seed=9, device=True)
    assert np.array_equal(xd.cpu().numpy().view(np.uint64), xb)


def test_probabilities_and_errors(rcs, ctx):
    text = config_qasm("c1")
    ref = oracle.build_state(text)
    st, psi = gpu_state(rcs, ctx, text)
    x = np.arange(0, 4096, 7, dtype=np.uint64)
    p = st.probabilities(x)
    xi = x.astype(np.int64)
    np.testing.assert_allclose(p, np.abs(psi[xi]) ** 2, rtol=1e-6, atol=0)        # |a|^2 of this state (fp64 of fp32)
    # vs the oracle: |p - p_o| <= (2|a| + d) d with the amplitude tolerance d = 1e-5
    assert (np.abs(p - np.abs(ref[xi]) ** 2) <= (2 * np.abs(ref[xi]) + 1e-5) * 1e-5).all()
    with pytest.raises(rcs.RcsError) as e:
        st.probabilities(np.array([4096], np.uint64))
    assert e.value.status == "RCS_ERR_SIZE"
    with pytest.raises(rcs.RcsError) as e:
        st.xeb(np.array([1, 1 << 12], np.uint64))
    assert e.value.status == "RCS_ERR_SIZE"


def test_memory_errors(rcs, ctx):
    import torch
    c = rcs.Circuit.from_qasm(config_qasm("c1"))
    small = torch.empty(100, dtype=torch.complex64, device="cuda")
    with pytest.raises(rcs.RcsError) as e:
        rcs.State.build(ctx, c, amps=small)
    assert e.value.status == "RCS_ERR_MEMORY" and e.value.bytes_required == 8 * 4096


def test_uniform_and_ideal_xeb_calibration(rcs, ctx):
    text = config_qasm("c2", n_qubits=20, rows=4, cols=5)
    st, _ = gpu_state(rcs, ctx, text)
    S = 200_000
    u = oracle.uniforms(5, S)
    xu = np.floor(u * (1 << 20)).astype(np.uint64)
    r = st.xeb(xu)
    assert abs(r["F"]) <= 5 * r["sigma"]
    r = st.xeb(st.sample(S, seed=6))
    assert abs(r["F"] - r["fstar"]) <= 5 * r["sigma"]


# ------------------------------------------------------------------ full size (BASELINE C3, bench launch config)
@pytest.mark.parametrize("k", [4, 6])
def test_full_size_c3_properties(rcs, ctx, k):
    """n = 32 (C3): oracle state is 64 GiB fp64, so parity at this size is checked by
    properties: norm, F* ~ 1 (Porter-Thomas), samples' XEB within 5 sigma of F*, and the
    circuit followed by its inverse returning e_0."""
    text = config_qasm("c3")
    c = rcs.Circuit.from_qasm(text)
    st = rcs.State.build(ctx, c, fuse_k=k)
    assert abs(st.norm - 1) <= 1e-5
    x = st.sample(1_000_000, seed=SHOT_SEED)
    r = st.xeb(x)
    assert abs(r["fstar"] - 1) < 0.05
    assert abs(r["F"] - r["fstar"]) <= 5 * r["sigma"]
    del st
    import torch
    torch.cuda.empty_cache()
    from tests.test_oracle_pins import inverse_qasm
    both = text + inverse_qasm(oracle.parse(text))
    st2 = rcs.State.build(ctx, rcs.Circuit.from_qasm(both), fuse_k=k)
    head = st2.copy_out(0, 1024)
    # C C^dagger = I: psi = e_0 within the amplitude tolerance, on the complex value (a phase
    # error fails), and the remaining mass 1 - |psi_0|^2 is the squared distance from e_0
    assert abs(complex(head[0]) - 1) <= 1e-5, head[0]
    assert abs(st2.norm - 1) <= 1e-5
    eps2 = max(0.0, st2.norm - abs(complex(head[0])) ** 2)
    assert eps2 <= 1e-10, eps2                    # ||psi - e_0||_2 <= 1e-5 (up to the norm drift)
    p = st2.probabilities(np.array([0, 1, 12345, (1 << 32) - 1], np.uint64))
    assert abs(p[0] - 1) < 2e-5 and p[1:].max() < 1e-10


# ------------------------------------------------------------------ precision over many passes
@pytest.mark.parametrize("tc_kernel", ["auto", "k9"])
def test_precision_over_120_passes_vs_oracle(rcs, ctx, tc_kernel):
    """>= 100 tensor-core passes stay within the BASELINE tolerance in amplitudes, in
    ||dpsi||_2 and in norm: the exact main term leaves no truncation bias (round 1's floating
    split drifted -1.4e-7 in norm^2 per pass and failed |T - 1| <= 1e-5 at ~70 passes)."""
    text = emit_qasm(generate(4, 5, 120, "ABCDCDAB", seed=21))
    st, psi = gpu_state(rcs, ctx, text, fuse_k=6, tc_kernel=tc_kernel)
    assert st.report["n_passes"] >= 100 and st.report["n_tc_passes"] == st.report["n_passes"]
    ref = oracle.build_state(text)
    check_amps(psi, ref)
    assert abs(st.norm - 1) <= 1e-5


def test_precision_circuit_then_inverse_n24(rcs, ctx):
    """C then C^dagger at n = 24 (4x6, 50 + 50 cycles, > 100 passes): psi = e_0 (closed form)."""
    from tests.test_oracle_pins import inverse_qasm
    text = emit_qasm(generate(4, 6, 50, "ABCDCDAB", seed=5))
    both = text + inverse_qasm(oracle.parse(text))
    st, psi = gpu_state(rcs, ctx, both, fuse_k=6)
    assert st.report["n_passes"] >= 100
    e0 = np.zeros_like(psi)
    e0[0] = 1
    assert np.linalg.norm(psi - e0) <= 1e-5
    assert abs(psi[0] - 1) <= 1e-5 and abs(st.norm - 1) <= 1e-5
