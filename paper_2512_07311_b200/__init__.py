"""B200-native exact state-vector RCS hot path (arXiv 2512.07311 problem statement).

Thin Python binding over librcs.so (include/rcs.h).  Every step of the path -- gate
fusion planning, state construction, remaps, sampling, XEB -- runs inside the library
(C++ host planner + sm_100a CUDA kernels + NCCL).  This module only marshals arguments;
PyTorch provides device memory, CUDA streams and the process group used to bootstrap NCCL.

    from paper_2512_07311_b200 import Circuit, Context, State
    c = Circuit.from_qasm(text)                      # PAPER §3.2 l.34
    ctx = Context()                                  # cuda:0, world 1  (or Context.from_process_group())
    st = State.build(ctx, c, fuse_k=4)               # PAPER §3.2 l.36
    x = st.sample(1_000_000, seed=2512)              # PAPER §3.2 l.38
    rep = st.xeb(x)                                  # PAPER §3.2 l.39, §5.1
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (REMAP_MODES, RcsError, check, lib, rcs_build_opts, rcs_build_report, rcs_circuit_counts,
                   rcs_error, rcs_plan_item, rcs_sample_report, rcs_xeb_report)

__all__ = ["Circuit", "Plan", "Context", "State", "RcsError", "lib", "sha256", "snapshot_info", "shard_shots",
           "job_seed", "xeb_from_probs"]

KIND_NAMES = {0: "sx", 1: "sy", 2: "sw", 3: "rz", 4: "fsim"}
ITEM_NAMES = {0: "pass", 1: "remap", 2: "swap"}


def _ptr(t):
    """Raw pointer of a torch tensor or numpy array."""
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


def _device_u64(ctx, x, what):
    """A caller CUDA tensor of bitstrings as the library reads it: contiguous 64-bit integers on
    the context's device (int64 / uint64 bit patterns); anything else is rejected."""
    import torch
    if x.dtype not in (torch.int64, torch.uint64):
        raise TypeError(f"{what}: bitstrings must be int64/uint64, got {x.dtype}")
    if x.device != torch.device("cuda", ctx.device):
        raise ValueError(f"{what}: tensor on {x.device}, context on cuda:{ctx.device}")
    return x.contiguous()


def _order_after_torch(ctx):
    """The library runs on ctx.stream: order it after the work torch queued on the current
    stream (allocations, producers of caller tensors)."""
    import torch
    ctx.stream.wait_stream(torch.cuda.current_stream(torch.device("cuda", ctx.device)))


def _order_torch_after(ctx):
    """Results the library wrote into torch tensors: later torch work on the current stream
    must follow the library's stream (the calls return after it drained; this also records
    the dependency for the caching allocator's stream bookkeeping)."""
    import torch
    torch.cuda.current_stream(torch.device("cuda", ctx.device)).wait_stream(ctx.stream)


class Circuit:
    """Parsed QASM circuit (host; rcs_circuit_load_qasm)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    @classmethod
    def from_qasm(cls, text: str) -> "Circuit":
        b = text.encode()
        h = C.c_void_p()
        err = rcs_error()
        check(lib().rcs_circuit_load_qasm(b, len(b), C.byref(h), C.byref(err)), err, "rcs_circuit_load_qasm")
        return cls(h.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().rcs_circuit_free(h)
            except Exception:   # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    def stats(self) -> dict:
        s = rcs_circuit_counts()
        check(lib().rcs_circuit_stats(self._h, C.byref(s)), None, "rcs_circuit_stats")
        return {f: getattr(s, f) for f, _ in s._fields_}

    @property
    def n_qubits(self) -> int:
        return self.stats()["n_qubits"]

    def gates(self) -> list:
        out = []
        k, q0, q1, m = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        th, ph = C.c_double(), C.c_double()
        for i in range(self.stats()["n_gates"]):
            check(lib().rcs_circuit_gate(self._h, i, C.byref(k), C.byref(q0), C.byref(q1), C.byref(th),
                                         C.byref(ph), C.byref(m)), None, "rcs_circuit_gate")
            qs = (q0.value,) if q1.value < 0 else (q0.value, q1.value)
            out.append((KIND_NAMES[k.value], qs, th.value, ph.value, m.value))
        return out


class Plan:
    """Host-only fused plan (rcs_plan_create): blocks, remaps, restore swaps."""

    def __init__(self, circuit: Circuit, fuse_k: int = 4, n_global: int = 0):
        self.circuit = circuit
        h = C.c_void_p()
        err = rcs_error()
        check(lib().rcs_plan_create(circuit._h, fuse_k, n_global, C.byref(h), C.byref(err)), err, "rcs_plan_create")
        self._h = h
        ni, npa, nr, ns, npf = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib().rcs_plan_summary(h, C.byref(ni), C.byref(npa), C.byref(nr), C.byref(ns))
        lib().rcs_plan_prefix(h, C.byref(npf))
        self.n_items, self.n_passes, self.n_remaps, self.n_swaps = ni.value, npa.value, nr.value, ns.value
        self.prefix = npf.value   # items [0, prefix): product-state prefix (disjoint blocks on |0...0>)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().rcs_plan_free(h)
            except Exception:   # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    def layout(self) -> dict:
        """restore_begin, final_pos (qubit -> physical position before the restore), initial_pos."""
        n = self.circuit.n_qubits
        rb = C.c_int()
        fp = (C.c_int * n)()
        ip = (C.c_int * n)()
        check(lib().rcs_plan_layout(self._h, C.byref(rb), fp, ip), None, "rcs_plan_layout")
        return {"restore_begin": rb.value, "final_pos": list(fp), "initial_pos": list(ip)}

    def items(self) -> list:
        out = []
        it = rcs_plan_item()
        for i in range(self.n_items):
            mat = np.zeros(2 * 4 ** 6, dtype=np.float64)
            check(lib().rcs_plan_item_get(self._h, i, C.byref(it), mat.ctypes.data_as(C.POINTER(C.c_double))),
                  None, "rcs_plan_item_get")
            d = {"type": ITEM_NAMES[it.type], "k": it.k}
            if it.type == 0:
                D = 1 << it.k
                d["qubits"] = list(it.qubits[:it.k])
                d["pos"] = list(it.pos[:it.k])
                d["n_gates"] = it.n_gates
                d["matrix"] = mat[:2 * D * D].view(np.complex128).reshape(D, D).copy()
            else:
                d["a"] = list(it.a[:it.k])
                d["b"] = list(it.b[:it.k])
            out.append(d)
        return out


class Context:
    """One per rank: device, CUDA stream and (world > 1) the NCCL communicator."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None, stream=None):
        import torch
        self.device = device
        self.rank, self.world = rank, world
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        h = C.c_void_p()
        err = rcs_error()
        idbuf = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id else None
        check(lib().rcs_context_create(device, rank, world, idbuf, C.c_void_p(self.stream.cuda_stream),
                                       C.byref(h), C.byref(err)), err, "rcs_context_create")
        self._h = h

    @classmethod
    def from_process_group(cls, device: int | None = None) -> "Context":
        """SPMD bootstrap over an initialised torch.distributed process group (any backend):
        rank 0 draws the NCCL unique id and broadcasts it."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = rank % max(1, torch.cuda.device_count())
        nid = None
        if world > 1:
            obj = [None]
            if rank == 0:
                n = lib().rcs_nccl_unique_id_bytes()
                buf = C.create_string_buffer(n)
                err = rcs_error()
                check(lib().rcs_nccl_unique_id(buf, C.byref(err)), err, "rcs_nccl_unique_id")
                obj = [bytes(buf.raw)]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        return cls(device, rank, world, nid)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().rcs_context_free(h)
            except Exception:   # interpreter shutdown: module globals already torn down
                pass
            self._h = None


class State:
    """A built state: amplitudes in a torch complex64 tensor owned by this object."""

    def __init__(self):
        self._h = None

    @classmethod
    def build(cls, ctx: Context, circuit: Circuit, fuse_k: int = 0, block_bits: int = 0, virtual_global: int = 0,
              timing: bool = False, staging_bytes: int = 0, amps=None, scratch=None,
              keep_layout: bool = False, remap_mode: str = "auto", overlap: bool = True, overlap_chunks: int = 0,
              overlap_sms: int = 0, tc_kernel: str = "auto", overlap_passes: int = 0,
              tc_schedule: str = "static", product_prefix: bool = True, tc_tma: str = "auto") -> "State":
        """rcs_state_build.  remap_mode: "auto" | "nccl" | "loopback" (world 1 + virtual_global: remaps
        through the NVLink peer-swap kernel between regions of this GPU); tc_kernel: "auto" | "k9" |
        "norow" (auto, but blocks on positions 0..5 on K9 instead of K12's row variant);
        tc_tma: "auto" (short K12 runs through tensor-map TMA) | "bulk" (one bulk copy per run)."""
        import torch
        n = circuit.n_qubits
        g = ctx.world.bit_length() - 1
        opts = rcs_build_opts(fuse_k, block_bits, virtual_global, 1 if timing else 0, staging_bytes,
                              1 if keep_layout else 0, REMAP_MODES[remap_mode], 0 if overlap else -1,
                              overlap_chunks, overlap_sms, {"auto": 0, "k9": 1, "norow": 2}[tc_kernel], overlap_passes,
                              0 if product_prefix else -1, {"static": 0, "dynamic": 1}[tc_schedule],
                              {"auto": 0, "bulk": -1}[tc_tma])
        sb = C.c_uint64()
        check(lib().rcs_state_scratch_bytes(ctx._h, circuit._h, C.byref(opts), C.byref(sb)), None,
              "rcs_state_scratch_bytes")
        dev = torch.device("cuda", ctx.device)
        if amps is None:
            amps = torch.empty(1 << (n - g), dtype=torch.complex64, device=dev)
        if scratch is None or scratch.numel() < sb.value:
            scratch = torch.empty(sb.value, dtype=torch.uint8, device=dev)
        self = cls()
        self.ctx, self.circuit, self.n, self.g = ctx, circuit, n, g
        self.amps, self.scratch = amps, scratch
        h = C.c_void_p()
        rep = rcs_build_report()
        err = rcs_error()
        _order_after_torch(ctx)   # torch's allocations / initialisation of amps and scratch
        check(lib().rcs_state_build(ctx._h, circuit._h, C.byref(opts), _ptr(amps), amps.numel() * 8, _ptr(scratch),
                                    scratch.numel(), C.byref(h), C.byref(rep), C.byref(err)), err, "rcs_state_build")
        self._h = h
        self.report = {f: getattr(rep, f) for f, _ in rep._fields_}
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().rcs_state_free(h)
            except Exception:   # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    def free(self):
        self.__del__()

    def canonicalize(self) -> None:
        """Collective: run the restore deferred by keep_layout=True (copy_out needs it)."""
        err = rcs_error()
        check(lib().rcs_state_canonicalize(self._h, C.byref(err)), err, "rcs_state_canonicalize")
        self.report["layout_kept"] = 0

    @property
    def norm(self) -> float:
        v = C.c_double()
        check(lib().rcs_state_norm(self._h, C.byref(v)), None, "rcs_state_norm")
        return v.value

    def pass_times(self) -> np.ndarray:
        n = C.c_int()
        lib().rcs_state_pass_times(self._h, None, 0, C.byref(n))
        out = np.zeros(n.value, dtype=np.float32)
        lib().rcs_state_pass_times(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), n.value, C.byref(n))
        return out

    def copy_out(self, first: int = None, count: int = None) -> np.ndarray:
        """complex64 amplitudes [first, first+count) (global logical index, this rank's shard)."""
        nl = self.n - self.g
        base = self.ctx.rank << nl
        first = base if first is None else first
        count = (1 << nl) - (first - base) if count is None else count
        out = np.empty(count, dtype=np.complex64)
        err = rcs_error()
        check(lib().rcs_state_copy_out(self._h, first, count, _ptr(out), C.byref(err)), err, "rcs_state_copy_out")
        return out

    def probabilities(self, x) -> np.ndarray:
        """|psi_x|^2 (host float64) of host bitstrings or a CUDA int64/uint64 tensor."""
        if hasattr(x, "data_ptr"):
            xa = _device_u64(self.ctx, x, "probabilities")
            _order_after_torch(self.ctx)   # the producer of x may still be queued on torch's stream
            n = xa.numel()
        else:
            xa = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
            n = xa.size
        p = np.empty(n, dtype=np.float64)
        err = rcs_error()
        check(lib().rcs_probabilities(self._h, _ptr(xa), n, _ptr(p), C.byref(err)), err, "rcs_probabilities")
        return p

    def sample(self, shots: int, seed: int = 2512, offset: int = 0, device: bool = False):
        """Bitstrings (uint64, qubit 0 = LSB) in shot order: numpy (host) or torch (device)."""
        import torch
        if device:
            out = torch.empty(shots, dtype=torch.int64, device=torch.device("cuda", self.ctx.device))
            _order_after_torch(self.ctx)   # the allocation may reuse memory torch's stream still uses
        else:
            out = np.empty(shots, dtype=np.uint64)
        rep = rcs_sample_report()
        err = rcs_error()
        check(lib().rcs_sample(self._h, shots, seed, offset, _ptr(out), C.byref(rep), C.byref(err)), err, "rcs_sample")
        if device:
            _order_torch_after(self.ctx)
        self.last_sample = {f: getattr(rep, f) for f, _ in rep._fields_}
        return out

    def sample_uniforms(self, u) -> np.ndarray:
        u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
        out = np.empty(u.size, dtype=np.uint64)
        rep = rcs_sample_report()
        err = rcs_error()
        check(lib().rcs_sample_uniforms(self._h, _ptr(u), u.size, _ptr(out), C.byref(rep), C.byref(err)), err,
              "rcs_sample_uniforms")
        return out

    # ---- paper stage 2: snapshot file (include/rcs.h rcs_snapshot_*)
    def save_snapshot(self, path: str) -> bytes:
        """Write the state atomically in the RCSS format; returns SHA-256(payload)."""
        dg = C.create_string_buffer(32)
        err = rcs_error()
        check(lib().rcs_snapshot_save(self._h, path.encode(), dg, C.byref(err)), err, "rcs_snapshot_save")
        return dg.raw

    @classmethod
    def load_snapshot(cls, ctx: "Context", path: str, block_bits: int = 0, amps=None, scratch=None) -> "State":
        """Digest-verified load of an RCSS file into a sample-ready single-GPU state."""
        import torch
        n = snapshot_info(path)["n_qubits"]
        sb = C.c_uint64()
        check(lib().rcs_snapshot_scratch_bytes(ctx._h, n, block_bits, C.byref(sb)), None,
              "rcs_snapshot_scratch_bytes")
        dev = torch.device("cuda", ctx.device)
        if amps is None:
            amps = torch.empty(1 << n, dtype=torch.complex64, device=dev)
        if scratch is None or scratch.numel() < sb.value:
            scratch = torch.empty(sb.value, dtype=torch.uint8, device=dev)
        self = cls()
        self.ctx, self.circuit, self.n, self.g = ctx, None, n, 0
        self.amps, self.scratch = amps, scratch
        h = C.c_void_p()
        err = rcs_error()
        _order_after_torch(ctx)
        check(lib().rcs_snapshot_load(ctx._h, path.encode(), block_bits, _ptr(amps), amps.numel() * 8,
                                      _ptr(scratch), scratch.numel(), C.byref(h), C.byref(err)), err,
              "rcs_snapshot_load")
        self._h = h
        self.report = {}
        return self

    def xeb(self, x) -> dict:
        """Linear XEB of host bitstrings or a CUDA int64/uint64 tensor against this state."""
        if not hasattr(x, "data_ptr"):
            x = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
            n = x.size
        else:
            x = _device_u64(self.ctx, x, "xeb")
            _order_after_torch(self.ctx)
            n = x.numel()
        rep = rcs_xeb_report()
        err = rcs_error()
        check(lib().rcs_xeb(self._h, _ptr(x), n, C.byref(rep), C.byref(err)), err, "rcs_xeb")
        return {f: getattr(rep, f) for f, _ in rep._fields_}


# ---- paper stages 2-4 helpers (host; include/rcs.h) ----------------------------------------
def sha256(data: bytes) -> bytes:
    out = C.create_string_buffer(32)
    check(lib().rcs_sha256(data, len(data), out), None, "rcs_sha256")
    return out.raw


def snapshot_info(path: str) -> dict:
    n = C.c_int()
    nb = C.c_uint64()
    dg = C.create_string_buffer(32)
    err = rcs_error()
    check(lib().rcs_snapshot_info(path.encode(), C.byref(n), C.byref(nb), dg, C.byref(err)), err,
          "rcs_snapshot_info")
    return {"n_qubits": n.value, "payload_bytes": nb.value, "digest": dg.raw}


def shard_shots(total: int, n_jobs: int) -> list:
    out = (C.c_uint64 * max(1, n_jobs))()
    check(lib().rcs_shard_shots(total, n_jobs, out), None, "rcs_shard_shots")
    return list(out)[:n_jobs]


def job_seed(base_seed: int, job_id: int) -> int:
    return int(lib().rcs_job_seed(base_seed, job_id))


def xeb_from_probs(n_qubits: int, p) -> dict:
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    rep = rcs_xeb_report()
    check(lib().rcs_xeb_from_probs(n_qubits, p.ctypes.data_as(C.POINTER(C.c_double)), p.size, C.byref(rep)), None,
          "rcs_xeb_from_probs")
    return {f: getattr(rep, f) for f, _ in rep._fields_}
