"""NumPy executor of the library's host plan (test infrastructure).

Runs the items returned by rcs_plan_item_get on a complex128 vector with plain index
arithmetic (no code shared with the CUDA kernels or the oracle):
  pass  -- v <- M v over every group differing only in physical bits pos[0..k)
  remap -- physical bits a[i] <-> b[i] swapped (single process: the whole vector)
  swap  -- the same on local bits
This checks the fuser (block matrices, order) and the remap/restore planner without a GPU.
"""
import numpy as np


def apply_block(psi: np.ndarray, M: np.ndarray, pos) -> None:
    n = psi.size.bit_length() - 1
    k = len(pos)
    # reshape so each target bit is its own axis; matrix bit i <-> pos[i]
    t = psi.reshape([2] * n)                  # axis a <-> bit (n-1-a)
    axes = [n - 1 - p for p in pos]           # matrix bit i -> tensor axis
    # move axes: matrix bit k-1 first ... bit 0 last, so flattening gives index sum b_i 2^i
    order = axes[::-1]
    rest = [a for a in range(n) if a not in order]
    tt = np.transpose(t, order + rest).reshape(1 << k, -1)
    tt = M @ tt
    inv = np.argsort(order + rest)
    psi[:] = np.transpose(tt.reshape([2] * n), inv).reshape(-1)


def bit_swap(psi: np.ndarray, pairs) -> None:
    n = psi.size.bit_length() - 1
    idx = np.arange(psi.size, dtype=np.int64)
    j = idx.copy()
    for a, b in pairs:
        ba = (idx >> a) & 1
        bb = (idx >> b) & 1
        diff = ba != bb
        j = np.where(diff, j ^ ((1 << a) | (1 << b)), j)
    psi[:] = psi[j]


def run_plan(items, n: int) -> np.ndarray:
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1
    for it in items:
        if it["type"] == "pass":
            apply_block(psi, it["matrix"], it["pos"])
        else:
            bit_swap(psi, list(zip(it["a"], it["b"])))
    return psi
