"""Seeded synthetic inputs (QASM circuits) shared by the oracle and the CUDA path.

Holds none of the method's arithmetic -- see gen.py."""
from .gen import (CONFIGS, SHOT_SEED, HEADLINE_SEED, SplitMix64, couplers, generate,
                  emit_qasm, config_qasm, random_qasm)

__all__ = ["CONFIGS", "SHOT_SEED", "HEADLINE_SEED", "SplitMix64", "couplers", "generate",
           "emit_qasm", "config_qasm", "random_qasm"]
