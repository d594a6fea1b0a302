"""The fp64 oracle on the full C4 circuit (2.5M shots), compared with the GPU path amplitude by
amplitude and shot by shot: no factorisation, no sampling of outputs -- every amplitude.

At n = 34 the oracle state needs 256 GiB of host memory and about an hour on 32 cores, more
than one gpurun call allows; `--n-qubits 33` truncates C4's 6x6 grid to 33 sites (2^33
amplitudes: 64-bit indexing, the same kernels and pass structure), which fits the 196 GiB /
16-core 1-GPU box in ~35 min (profiles/r02/oracle_full/).  A one-off evidence run, not a
pytest case.  Steps:

  1. GPU (the bench's default options, fuse_k 6): build, T, sample 2.5M shots with the bench's
     seed, XEB and F* -- the state stays resident on the device (128 GiB).
  2. Oracle (timed phase by phase -> a MEASURED full-workload CPU baseline): parse, build the
     complex128 state, T, sample the same uniforms, XEB of its own shots and of the GPU's.
  3. Compare on the device, 2^26 amplitudes at a time: max |d psi|, ||d psi||_2 (north_star:
     <= 1e-5), then every shot: identical picks, or the G17 excuse (t_s within 1e-6 of the
     separating boundary of the oracle's CDF, evaluated exactly at the GPU's pick), and the
     normalised-CDF excess of each GPU pick.  XEB: same-sample |F_gpu - F_oracle| (<= 1e-3).

    python scripts/oracle_c4_full.py --n-qubits 33 --out gpurun_out/oracle_full
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/oracle_full")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--shots", type=int, default=2_500_000)
    ap.add_argument("--n-qubits", type=int, default=0, help="truncate the config's grid to this many qubits")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    logf = open(os.path.join(a.out, "log.txt"), "w")

    def log(s):
        print(s, flush=True)
        logf.write(s + "\n")
        logf.flush()

    import torch
    import oracle
    import paper_2512_07311_b200 as rcs
    from rcs_workload import SHOT_SEED, config_qasm
    text = config_qasm(a.config, **({"n_qubits": a.n_qubits} if a.n_qubits else {}))
    S = a.shots
    R = {"config": a.config, "shots": S, "host_cores": os.cpu_count()}
    mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    need = 16 * (1 << (a.n_qubits or {"c4": 34, "c5": 36}.get(a.config, 0))) + (24 << 30)
    R["host_mem_gib"] = mem / 2 ** 30
    if mem < need:
        log(f"host RAM {mem / 2**30:.1f} GiB < {need / 2**30:.1f} GiB needed: not run")
        sys.exit(3)

    # 1. GPU
    ctx = rcs.Context(0)
    c = rcs.Circuit.from_qasm(text)
    n = c.n_qubits
    R["n"] = n
    t0 = time.time()
    st = rcs.State.build(ctx, c, fuse_k=6)
    T_gpu = st.norm
    x_g = st.sample(S, seed=SHOT_SEED)
    xr = st.xeb(x_g)
    R["gpu"] = {"wall_s": time.time() - t0, "n_passes": st.report["n_passes"], "n_prefix": st.report["n_prefix"],
                "T_minus_1": T_gpu - 1, "F": xr["F"], "sigma": xr["sigma"], "fstar": xr["fstar"]}
    log(f"gpu: {R['gpu']}")

    # 2. oracle, timed
    oracle.set_num_threads(os.cpu_count())
    R["oracle_threads"] = oracle.num_threads()
    t0 = time.time()
    oc = oracle.parse(text)
    t_parse = time.time() - t0
    t0 = time.time()
    ref = oc.build_state()
    t_build = time.time() - t0
    log(f"oracle build: {t_build:.1f} s ({R['oracle_threads']} threads)")
    u = oracle.uniforms(SHOT_SEED, S)
    t0 = time.time()
    x_o, T_o = oracle.sample(ref, u, norm_tol=1e-6)
    t_sample = time.time() - t0
    t0 = time.time()
    F_o, s_o, _ = oracle.xeb(ref, x_o)
    t_xeb = time.time() - t0
    F_og, _, _ = oracle.xeb(ref, x_g)          # same-sample: the oracle's p at the GPU's shots
    fstar_o = oracle.fstar(ref)
    R["oracle"] = {"parse_s": t_parse, "build_s": t_build, "sample_s": t_sample, "xeb_s": t_xeb,
                   "step_s": t_parse + t_build + t_sample + t_xeb, "T_minus_1": T_o - 1, "F": F_o, "sigma": s_o,
                   "F_on_gpu_shots": F_og, "fstar": fstar_o}
    log(f"oracle: {R['oracle']}")

    # 3a. amplitudes, on the device
    dev = st.amps.device
    amps = st.amps.view(-1)
    chunk = 1 << 26
    maxd, ss = 0.0, 0.0
    t0 = time.time()
    for a0 in range(0, 1 << n, chunk):
        r = torch.from_numpy(ref[a0:a0 + chunk]).to(dev)
        d = amps[a0:a0 + chunk].to(torch.complex128) - r
        maxd = max(maxd, d.abs().max().item())
        ss += (d.real.square() + d.imag.square()).sum().item()
        del r, d
    eps = math.sqrt(ss)
    R["amps"] = {"max_abs_d": maxd, "eps_l2": eps, "compare_s": time.time() - t0}
    log(f"amps: {R['amps']}")

    # 3b. shots: the oracle's exact sequential CDF evaluated at the GPU's picks
    xg = x_g.astype(np.int64)
    order = np.argsort(xg, kind="stable")
    xs = xg[order]
    C_hi = np.empty(S)
    C_lo = np.empty(S)
    run = 0.0
    j = 0
    for a0 in range(0, 1 << n, chunk):
        p = ref[a0:a0 + chunk].real ** 2 + ref[a0:a0 + chunk].imag ** 2
        cs = np.cumsum(p)
        cs += run
        k = np.searchsorted(xs, a0 + chunk, side="left")
        idx = xs[j:k] - a0
        C_hi[order[j:k]] = cs[idx]
        C_lo[order[j:k]] = np.where(idx > 0, cs[np.maximum(idx - 1, 0)], run)
        run = cs[-1]
        j = k
    t = u * T_o
    bad = ~((t >= C_lo - 1e-6) & (t <= C_hi + 1e-6))
    excess = np.maximum(C_lo / T_o - u, 0.0) + np.maximum(u - C_hi / T_o, 0.0)
    R["shots"] = {"identical": int((x_o == x_g).sum()), "differ": int((x_o != x_g).sum()),
                  "unexcused_g17": int(bad.sum()), "max_excess_normalised": float(excess.max())}
    R["xeb"] = {"F_gpu": xr["F"], "F_oracle_same_sample": F_og, "abs_diff": abs(xr["F"] - F_og),
                "fstar_gpu": xr["fstar"], "fstar_oracle": fstar_o}
    ok = (maxd <= 1e-5 and eps <= 1e-5 and abs(T_gpu - 1) <= 1e-5 and int(bad.sum()) == 0
          and abs(xr["F"] - F_og) <= 1e-3)
    R["pass"] = bool(ok)
    log(f"shots: {R['shots']}")
    log(f"xeb: {R['xeb']}")
    log(f"PASS={ok}")
    with open(os.path.join(a.out, f"oracle_{a.config}_n{n}_full.json"), "w") as f:
        json.dump(R, f, indent=1)
    st.free()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
