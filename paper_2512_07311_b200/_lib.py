"""ctypes declarations mirroring include/rcs.h exactly (argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librcs.so")

STATUS = {0: "RCS_OK", 1: "RCS_ERR_PARSE", 2: "RCS_ERR_UNKNOWN_GATE", 3: "RCS_ERR_QUBIT_RANGE",
          4: "RCS_ERR_ARITY", 5: "RCS_ERR_MEMORY", 6: "RCS_ERR_NORM", 7: "RCS_ERR_SIZE",
          8: "RCS_ERR_ARG", 9: "RCS_ERR_CUDA", 10: "RCS_ERR_NCCL", 11: "RCS_ERR_IO", 12: "RCS_ERR_FORMAT",
          13: "RCS_ERR_DIGEST"}


class rcs_error(C.Structure):
    _fields_ = [("code", C.c_int), ("line", C.c_int), ("col", C.c_int),
                ("bytes_required", C.c_uint64), ("msg", C.c_char * 256)]


class rcs_circuit_counts(C.Structure):
    _fields_ = [(f, C.c_int) for f in ("n_qubits", "n_moments", "n_gates", "n_measure",
                                       "n_sx", "n_sy", "n_sw", "n_rz", "n_fsim")]


# rcs_build_opts.remap_mode
REMAP_MODES = {"auto": 0, "nccl": 1, "loopback": 2}


class rcs_build_opts(C.Structure):
    _fields_ = [("fuse_k", C.c_int), ("block_bits", C.c_int), ("virtual_global", C.c_int),
                ("timing", C.c_int), ("staging_bytes", C.c_uint64), ("keep_layout", C.c_int),
                ("remap_mode", C.c_int), ("overlap", C.c_int), ("overlap_chunks", C.c_int),
                ("overlap_sms", C.c_int), ("tc_kernel", C.c_int), ("overlap_passes", C.c_int),
                ("product_prefix", C.c_int), ("tc_schedule", C.c_int), ("tc_tma", C.c_int)]


class rcs_build_report(C.Structure):
    _fields_ = [("n_passes", C.c_int), ("n_remaps", C.c_int), ("n_swaps", C.c_int), ("fuse_k", C.c_int),
                ("plan_ms", C.c_double), ("build_ms", C.c_double), ("pass_ms", C.c_double),
                ("pass_ms_min", C.c_double), ("pass_ms_max", C.c_double), ("remap_ms", C.c_double),
                ("blocksum_ms", C.c_double), ("pass_bytes", C.c_uint64), ("remap_bytes", C.c_uint64),
                ("norm", C.c_double), ("n_tc_passes", C.c_int), ("swap_ms", C.c_double),
                ("layout_kept", C.c_int), ("n_pipelined", C.c_int), ("n_peer_remaps", C.c_int),
                ("remap_kernel_ms", C.c_double), ("n_prefix", C.c_int), ("prefix_ms", C.c_double),
                ("upload_bytes", C.c_uint64)]


class rcs_sample_report(C.Structure):
    _fields_ = [("shots", C.c_uint64), ("total_prob", C.c_double), ("sample_ms", C.c_double)]


class rcs_xeb_report(C.Structure):
    _fields_ = [("n_qubits", C.c_int), ("shots", C.c_uint64), ("F", C.c_double), ("sigma", C.c_double),
                ("mean_p", C.c_double), ("fstar", C.c_double)]


class rcs_plan_item(C.Structure):
    _fields_ = [("type", C.c_int), ("k", C.c_int), ("qubits", C.c_int * 8), ("pos", C.c_int * 8),
                ("a", C.c_int * 8), ("b", C.c_int * 8), ("n_gates", C.c_int)]


# name -> (restype, argtypes); every symbol include/rcs.h declares
VP = C.c_void_p
PP = C.POINTER(C.c_void_p)
E = C.POINTER(rcs_error)
U64P = C.POINTER(C.c_uint64)
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)
SIGNATURES = {
    "rcs_status_string": (C.c_char_p, [C.c_int]),
    "rcs_kernel_launches": (C.c_uint64, []),
    "rcs_circuit_load_qasm": (C.c_int, [C.c_char_p, C.c_size_t, PP, E]),
    "rcs_circuit_stats": (C.c_int, [VP, C.POINTER(rcs_circuit_counts)]),
    "rcs_circuit_gate": (C.c_int, [VP, C.c_int, IP, IP, IP, DP, DP, IP]),
    "rcs_circuit_free": (None, [VP]),
    "rcs_plan_create": (C.c_int, [VP, C.c_int, C.c_int, PP, E]),
    "rcs_plan_summary": (C.c_int, [VP, IP, IP, IP, IP]),
    "rcs_plan_prefix": (C.c_int, [VP, IP]),
    "rcs_plan_item_get": (C.c_int, [VP, C.c_int, C.POINTER(rcs_plan_item), DP]),
    "rcs_plan_free": (None, [VP]),
    "rcs_plan_layout": (C.c_int, [VP, IP, IP, IP]),
    "rcs_nccl_unique_id_bytes": (C.c_int, []),
    "rcs_nccl_unique_id": (C.c_int, [VP, E]),
    "rcs_context_create": (C.c_int, [C.c_int, C.c_int, C.c_int, VP, VP, PP, E]),
    "rcs_context_free": (None, [VP]),
    "rcs_state_scratch_bytes": (C.c_int, [VP, VP, C.POINTER(rcs_build_opts), U64P]),
    "rcs_state_build": (C.c_int, [VP, VP, C.POINTER(rcs_build_opts), VP, C.c_uint64, VP, C.c_uint64, PP,
                                  C.POINTER(rcs_build_report), E]),
    "rcs_state_canonicalize": (C.c_int, [VP, E]),
    "rcs_state_pass_times": (C.c_int, [VP, C.POINTER(C.c_float), C.c_int, IP]),
    "rcs_state_norm": (C.c_int, [VP, DP]),
    "rcs_state_copy_out": (C.c_int, [VP, C.c_uint64, C.c_uint64, VP, E]),
    "rcs_probabilities": (C.c_int, [VP, VP, C.c_uint64, VP, E]),
    "rcs_sample": (C.c_int, [VP, C.c_uint64, C.c_uint64, C.c_uint64, VP, C.POINTER(rcs_sample_report), E]),
    "rcs_sample_uniforms": (C.c_int, [VP, VP, C.c_uint64, VP, C.POINTER(rcs_sample_report), E]),
    "rcs_xeb": (C.c_int, [VP, VP, C.c_uint64, C.POINTER(rcs_xeb_report), E]),
    "rcs_state_free": (None, [VP]),
    "rcs_sha256": (C.c_int, [VP, C.c_uint64, VP]),
    "rcs_snapshot_save": (C.c_int, [VP, C.c_char_p, VP, E]),
    "rcs_snapshot_info": (C.c_int, [C.c_char_p, IP, U64P, VP, E]),
    "rcs_snapshot_scratch_bytes": (C.c_int, [VP, C.c_int, C.c_int, U64P]),
    "rcs_snapshot_load": (C.c_int, [VP, C.c_char_p, C.c_int, VP, C.c_uint64, VP, C.c_uint64, PP, E]),
    "rcs_shard_shots": (C.c_int, [C.c_uint64, C.c_int, U64P]),
    "rcs_job_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "rcs_xeb_from_probs": (C.c_int, [C.c_int, DP, C.c_uint64, C.POINTER(rcs_xeb_report)]),
}

_lib = None


class RcsError(RuntimeError):
    def __init__(self, code, err: rcs_error | None = None, where: str = ""):
        self.code = code
        self.status = STATUS.get(code, str(code))
        self.line = err.line if err is not None else 0
        self.col = err.col if err is not None else 0
        self.bytes_required = err.bytes_required if err is not None else 0
        msg = err.msg.decode(errors="replace") if err is not None else ""
        super().__init__(f"{where}: {self.status}: {msg}" + (f" (line {self.line}, col {self.col})" if self.line else ""))


def lib():
    """Load librcs.so (built in-tree by paper_2512_07311_b200.build).  No fallback: a missing
    or unloadable library raises."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2512_07311_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code, err=None, where=""):
    if code != 0:
        raise RcsError(code, err, where)
