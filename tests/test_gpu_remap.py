"""The multi-GPU remap data path on ONE GPU (loopback): driver-visible parity for k_peer_swap.

With remap_mode="loopback" and virtual_global=g the state buffer is treated as 2^g virtual
ranks' shards (consecutive regions; rank r holds logical indices [r 2^(n-g), (r+1) 2^(n-g)) as
in DESIGN.md §7) and every REMAP item runs through the NVLink peer-swap kernel (k_peer_swap)
with the other regions as peers -- sequentially, or pipelined with the neighbouring
tensor-core passes exactly as between GPUs.  The fused arithmetic is
P-independent, so the state must equal the single-shard build bit for bit, and the oracle
within the BASELINE tolerance (§3.2 l.36: the state is constructed exactly).
"""
import numpy as np
import pytest

import oracle
from rcs_workload import SHOT_SEED, config_qasm, emit_qasm, generate

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


CASES = {
    "grid20_k4": (emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=3)), 4),
    "grid20_k6": (emit_qasm(generate(4, 5, 16, "ABCDCDAB", seed=3)), 6),
    "c2_k6": (config_qasm("c2"), 6),
    # a block on positions 0..5 (K12's row variant), also inside pipelined (chunked) passes
    "row21_k6": (emit_qasm(generate(3, 7, 12, "ABCDCDAB", seed=1)), 6),
}


def check_amps(psi, ref):
    d = psi.astype(np.complex128) - ref
    assert np.abs(d).max() <= 1e-5 and np.linalg.norm(d) <= 1e-5


# pipelining: "chain" = the default (up to 3 passes after a remap run chunk by chunk behind its
# swaps), "next" = only the pass right after the remap, "off" = sequential remaps
OVERLAP = {"chain": {}, "next": {"overlap_passes": 1}, "off": {"overlap": False}}


@pytest.mark.parametrize("mode", list(OVERLAP))
@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("case", list(CASES))
def test_loopback_remaps_bitwise(rcs, ctx, case, g, mode):
    text, k = CASES[case]
    overlap = mode != "off"
    c = rcs.Circuit.from_qasm(text)
    single = rcs.State.build(ctx, c, fuse_k=k)
    psi1 = single.copy_out()
    x1 = single.sample(50_000, seed=SHOT_SEED)
    single.free()
    st = rcs.State.build(ctx, c, fuse_k=k, virtual_global=g, remap_mode="loopback", timing=True, **OVERLAP[mode])
    rep = st.report
    assert rep["n_remaps"] > 0 and rep["n_peer_remaps"] > 0, rep
    if k == 6 and overlap:
        assert rep["n_pipelined"] > 0, rep          # chunked swaps overlapped with pass chunks
    if not overlap or k == 4:
        assert rep["n_pipelined"] == 0, rep
    assert rep["n_passes"] == len(st.pass_times())
    assert rep["remap_bytes"] > 0 and rep["remap_kernel_ms"] > 0, rep
    psi = st.copy_out()
    assert np.array_equal(psi, psi1), case        # P-invariance through the peer-swap path
    check_amps(psi, oracle.build_state(text))
    assert np.array_equal(st.sample(50_000, seed=SHOT_SEED), x1)


@pytest.mark.parametrize("g", [2, 3])
def test_loopback_keep_layout_and_canonicalize(rcs, ctx, g):
    """keep_layout with loopback remaps: same shots as the canonical build; canonicalize() runs
    the deferred restore through the peer-swap kernel."""
    text, k = CASES["c2_k6"]
    c = rcs.Circuit.from_qasm(text)
    can = rcs.State.build(ctx, c, fuse_k=k, virtual_global=g)
    kept = rcs.State.build(ctx, c, fuse_k=k, virtual_global=g, remap_mode="loopback", keep_layout=True)
    assert kept.report["layout_kept"] == 1
    assert np.array_equal(can.sample(100_000, seed=SHOT_SEED), kept.sample(100_000, seed=SHOT_SEED))
    kept.canonicalize()
    assert np.array_equal(kept.copy_out(), can.copy_out())


def test_loopback_option_errors(rcs, ctx):
    c = rcs.Circuit.from_qasm(CASES["grid20_k4"][0])
    with pytest.raises(rcs.RcsError) as e:
        rcs.State.build(ctx, c, remap_mode="loopback")            # needs virtual_global >= 1
    assert e.value.status == "RCS_ERR_ARG"
    with pytest.raises(rcs.RcsError) as e:
        rcs.State.build(ctx, c, virtual_global=4, remap_mode="loopback")   # at most 8 virtual ranks
    assert e.value.status == "RCS_ERR_ARG"
