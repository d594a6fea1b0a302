"""Sustained-load probe: HBM rate, SM clock and board power for
  copy   : torch in-place x.mul_(1) over a 64 GiB complex64 buffer (read+write, the pass's traffic)
  pass   : the library's C4 build (36 tensor-core passes)
Each experiment runs ~3 s; nvidia-smi is sampled every 100 ms meanwhile.
usage: python scripts/power_probe.py copy|pass
"""
import os
import statistics
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def sampler():
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
    return p, f


def stop(p, f):
    time.sleep(0.2)
    p.terminate()
    p.wait()
    rows = [ln.split(",") for ln in open(f.name) if ln.count(",") >= 2]
    sm = [float(r[0]) for r in rows]
    pw = [float(r[1]) for r in rows]
    tp = [float(r[2]) for r in rows]
    return sm, pw, tp


def main():
    import torch
    what = sys.argv[1]
    if what == "copy":
        x = torch.zeros(1 << 33, dtype=torch.complex64, device="cuda")   # 64 GiB
        nbytes = 2 * x.numel() * 8
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
        p, f = sampler()
        for a, b in ev:
            a.record()
            x.mul_(1.0)
            b.record()
        torch.cuda.synchronize()
        sm, pw, tp = stop(p, f)
        ms = [a.elapsed_time(b) for a, b in ev]
        gbs = [nbytes / (m / 1e3) / 1e9 for m in ms]
        print(f"copy: GB/s first {gbs[0]:.0f} median {statistics.median(gbs):.0f} last10 {statistics.median(gbs[-10:]):.0f}"
              f" | sm MHz median {statistics.median(sm):.0f} min {min(sm):.0f} | W max {max(pw):.0f} median"
              f" {statistics.median(pw):.0f} | temp {max(tp):.0f}")
    else:
        import paper_2512_07311_b200 as rcs
        from rcs_workload import config_qasm
        ctx = rcs.Context(0)
        c = rcs.Circuit.from_qasm(config_qasm("c4"))
        amps = torch.empty(1 << 34, dtype=torch.complex64, device="cuda")
        st = rcs.State.build(ctx, c, fuse_k=6, amps=amps)    # warm (plan + operands cached)
        scratch = st.scratch
        st.free()
        p, f = sampler()
        allg = []
        for _ in range(2):
            st = rcs.State.build(ctx, c, fuse_k=6, timing=True, amps=amps, scratch=scratch)
            allg += [16 * (1 << 34) / (m / 1e3) / 1e9 for m in st.pass_times()]
            st.free()
        sm, pw, tp = stop(p, f)
        print(f"pass: GB/s first10 {statistics.median(allg[:10]):.0f}"
              f" median {statistics.median(allg):.0f} last20 {statistics.median(allg[-20:]):.0f}"
              f" | sm MHz median {statistics.median(sm):.0f} min {min(sm):.0f} | W max {max(pw):.0f} median"
              f" {statistics.median(pw):.0f} | temp {max(tp):.0f}")


if __name__ == "__main__":
    main()
