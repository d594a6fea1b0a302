"""fp64 CPU oracle for the RCS hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  The product package never imports it.
See rcs_oracle.c for what each function follows in the paper.
"""
from .oracle import (Oracle, OracleError, build_oracle, parse, gate_matrix, apply_gate,
                     build_state, total_prob, uniforms, sample, xeb, fstar, num_threads,
                     set_num_threads)

__all__ = ["Oracle", "OracleError", "build_oracle", "parse", "gate_matrix", "apply_gate",
           "build_state", "total_prob", "uniforms", "sample", "xeb", "fstar", "num_threads",
           "set_num_threads"]
