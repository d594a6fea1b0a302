"""Per-pass SM clock and board power during a C4 build (why the live pass rate sits below the
ncu-isolated one): NVML sampled every ~2 ms in a thread, pass windows placed by the
device-timed pass durations (passes run back to back on one stream).

    python scripts/pass_power_trace.py [--config c4] [--builds 3] [--out profiles/...txt]
"""
import argparse
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--builds", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import pynvml
    import torch
    import paper_2512_07311_b200 as rcs
    from rcs_workload import config_qasm
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples = []
    stop = threading.Event()

    def poll():
        while not stop.is_set():
            t = time.perf_counter()
            samples.append((t, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.002)

    th = threading.Thread(target=poll, daemon=True)
    th.start()
    ctx = rcs.Context(0)
    c = rcs.Circuit.from_qasm(config_qasm(a.config))
    lines = []
    bufs = {}
    for b in range(a.builds):
        torch.cuda.synchronize()
        st = rcs.State.build(ctx, c, fuse_k=6, timing=True, **bufs)   # reuse the 128 GiB buffers
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        pt = st.pass_times()
        bufs = {"amps": st.amps, "scratch": st.scratch}
        st.free()
        if b != a.builds - 1:
            continue
        S = np.array(samples)
        ends = t_end - (pt[::-1].cumsum()[::-1] - pt) / 1e3     # pass i ends at t_end - sum(later passes)
        starts = ends - pt / 1e3
        lines.append(f"# {a.config}: pass, ms, GB/s, SM MHz (median in window), board W (median), samples")
        per = 16.0 * (1 << c.n_qubits)
        for i, (s0, s1, ms) in enumerate(zip(starts, ends, pt)):
            w = S[(S[:, 0] >= s0) & (S[:, 0] <= s1)]
            mhz = float(np.median(w[:, 1])) if len(w) else float("nan")
            pw = float(np.median(w[:, 2])) if len(w) else float("nan")
            lines.append(f"{i:3d} {ms:8.2f} {per / ms / 1e6:7.0f} {mhz:7.0f} {pw:7.0f} {len(w):4d}")
        ms = np.array(pt)
        mhzs = np.array([float(l.split()[3]) for l in lines[1:]])
        ok = np.isfinite(mhzs)
        if ok.sum() > 3:
            r = np.corrcoef(1 / ms[ok], mhzs[ok])[0, 1]
            lines.append(f"# corr(pass rate, SM clock) = {r:.3f}; mean rate {per / ms.mean() / 1e6:.0f} GB/s")
    stop.set()
    th.join()
    print("\n".join(lines))
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
