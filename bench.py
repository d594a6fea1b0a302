#!/usr/bin/env python
"""Benchmark of the RCS hot path (BASELINE.json metric: "fused gate-pass HBM GB/s vs peak;
circuit build s; shots/sec; XEB at 1/2/4/8 B200").

One step = the whole hot path on one synthetic input: build the exact complex64 state of the
BASELINE config-4 circuit (n=34, 6x6 grid truncated, 20 cycles ABCDCDAB, seed 1) by fused
dense gate passes (+ NCCL remaps when sharded), sample 2.5M shots (shot seed 2512), score
linear XEB.  The same workload runs at every N (strong scaling; the state is sharded over the
top log2(N) qubits).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

value  = gate-pass algorithmic bytes of all ranks (16 B per amplitude per fused pass)
         x K / max-over-ranks device time of the K timed steps  [GB/s]
e2e    = the same through the public API with host buffers (QASM text in, bitstrings out to
         host, XEB scored from the host array), copies inside the timed region.
--impl reference runs the fp64 CPU oracle (the only other place bench.py executes oracle/).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from rcs_workload import CONFIGS, SHOT_SEED, config_qasm  # noqa: E402

METRIC = "fused gate-pass HBM GB/s (whole RCS step: state build + shots + XEB)"

# Fused passes per config and fuse_k of the library's planner (P-independent).  The reference
# arm converts oracle time into the same unit with this table instead of calling our engine;
# tests/test_bench.py keeps it equal to rcs_plan_create's output.
# leading blocks written as a product state (rcs_plan_prefix: one write-only kernel replaces the
# state initialisation and these passes), likewise kept equal to the planner
PLAN_PREFIX = {'c1': {3: 4, 4: 2, 5: 2, 6: 2},
               'c2': {3: 8, 4: 6, 5: 5, 6: 4},
               'c3': {3: 11, 4: 8, 5: 7, 6: 6},
               'c4': {3: 12, 4: 9, 5: 6, 6: 6},
               'c5': {3: 12, 4: 8, 5: 6, 6: 6},
               'w33': {3: 11, 4: 9, 5: 7, 6: 6},
               'w35': {3: 6, 4: 8, 5: 5, 6: 6}}
PLAN_PASSES = {'c1': {3: 32, 4: 19, 5: 14, 6: 8},
               'c2': {3: 98, 4: 45, 5: 38, 6: 27},
               'c3': {3: 102, 4: 56, 5: 44, 6: 33},
               'c4': {3: 143, 4: 76, 5: 55, 6: 36},
               'c5': {3: 157, 4: 82, 5: 63, 6: 36},
               'w33': {3: 119, 4: 74, 5: 53, 6: 39},
               'w35': {3: 142, 4: 83, 5: 52, 6: 46}}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fuse-k", type=int, default=6)
    ap.add_argument("--shots", type=int, default=0, help="override the config's shot count")
    ap.add_argument("--e2e-steps", type=int, default=-1, help="default: --steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--canonical", action="store_true", help="restore the canonical layout after every build")
    ap.add_argument("--no-overlap", action="store_true", help="sequential remaps (no pipelining with the passes)")
    ap.add_argument("--overlap-passes", type=int, default=0, help="passes after a remap pipelined behind it (0: default)")
    ap.add_argument("--dynamic-tiles", action="store_true", help="K12 dynamic tile scheduler (default: static)")
    ap.add_argument("--overlap-sms", type=int, default=0, help="SMs left to the pipelined swaps (0: default)")
    ap.add_argument("--overlap-chunks", type=int, default=0, help="pipelined remaps: 2^k chunks (0: default 2)")
    ap.add_argument("--no-prefix", action="store_true", help="run the product-state prefix blocks as passes")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    return ap.parse_args()


def workload(args):
    cfg = dict(CONFIGS[args.config])
    shots = args.shots or cfg["shots"]
    desc = (f"{args.config}: n={cfg['n_qubits']} ({cfg['rows']}x{cfg['cols']} grid"
            f"{' truncated' if cfg['n_qubits'] < cfg['rows'] * cfg['cols'] else ''}), {cfg['cycles']} cycles "
            f"{cfg['pattern']}, {shots} shots")
    return cfg, shots, desc


# ----------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for ln in fh:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1])]
        mx = max((num(r[2]) for r in rows if num(r[2])), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max((num(r[3]) or 0 for r in rows), default=None)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def host_info():
    """Host the oracle baseline runs on (nproc, CPU model/sockets, memory)."""
    info = {"nproc": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal:"):
                    info["mem_total_gib"] = round(int(ln.split()[1]) / 2 ** 20, 1)
    except Exception:
        pass
    return info


def ncu_traffic(config, world):
    """Per-launch DRAM bytes of the gate-pass kernel from a committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{config}/N{world}")
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_sample(cfg_name: str, cfg: dict, shots: int, budget_s: float, n_small: int = 28):
    """Bounded oracle run on the host cores, projected to the full workload.

    Sample: the first G gates of the same generator config restricted to n_small qubits
    (same grid, truncated row-major), timed build; plus sampling + XEB of min(shots, 250k)
    shots on that state.  Projection: build time scales with 2^n * gates (per-gate sweeps),
    sampling with 2^n (one streaming CDF pass) -- both linear, as in the oracle's code."""
    import oracle
    # all host cores, also under torchrun (which exports OMP_NUM_THREADS=1 to every rank)
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    n_small = min(n_small, cfg["n_qubits"])
    text = config_qasm(cfg_name, n_qubits=n_small)
    full_gates = len(oracle.parse(config_qasm(cfg_name)).gates)
    circ = oracle.parse(text)
    # calibrate G so that the build takes ~budget/2: per-gate cost from the difference of a 2- and
    # a 6-gate build (the first build_state also allocates and zeroes the 2^n state)
    def timed(g):
        t0 = time.perf_counter()
        circ.build_state(max_gates=g)
        return time.perf_counter() - t0
    timed(2)               # first touch of the state's pages
    t2 = timed(2)
    t6 = timed(6)
    per_gate = max((t6 - t2) / 4, 1e-4)
    fixed = max(0.0, t2 - 2 * per_gate)
    G = max(6, min(len(circ.gates), int(budget_s * 0.5 / per_gate)))
    t0 = time.perf_counter()
    psi = circ.build_state(max_gates=G)
    t_build = time.perf_counter() - t0
    S = min(shots, 250_000)
    u = oracle.uniforms(SHOT_SEED, S)
    t0 = time.perf_counter()
    x, _ = oracle.sample(psi, u, norm_tol=1e-6)
    oracle.xeb(psi, x)
    t_samp = time.perf_counter() - t0
    n_full = cfg["n_qubits"]
    scale = 2.0 ** (n_full - n_small)
    proj = max(t_build - fixed, 1e-9) / G * full_gates * scale + t_samp * scale
    host = host_info()
    need_gib = 16 * 2 ** n_full / 2 ** 30
    desc = (f"oracle fp64, first {G} of {len(circ.gates)} gates of the {cfg_name} circuit at n={n_small} "
            f"({t_build:.2f} s) + sample/XEB of {S} shots ({t_samp:.2f} s); projected linearly in 2^n*gates "
            f"to n={n_full}, {full_gates} gates, {shots} shots: {proj:.1f} s (projected, not run in full: the "
            f"fp64 state needs {need_gib:.0f} GiB, host RAM {host.get('mem_total_gib', '?')} GiB, and a full run "
            f"takes ~{proj / 60:.0f} min)")
    return proj, desc, oracle.num_threads(), t_build + t_samp


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2512_07311_b200 as rcs
    from paper_2512_07311_b200._lib import rcs_sample_report, rcs_error, check

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        ctx = rcs.Context.from_process_group(local)
    else:
        ctx = rcs.Context(local)
    L = rcs.lib()
    cfg, shots, desc = workload(args)
    text = config_qasm(args.config)
    circuit = rcs.Circuit.from_qasm(text)
    n = cfg["n_qubits"]
    g = world.bit_length() - 1
    plan = rcs.Plan(circuit, args.fuse_k, g)
    amps = torch.empty(1 << (n - g), dtype=torch.complex64, device=dev)
    keep = not args.canonical   # skip the final layout restore: samples/XEB are layout-independent
    bopts = {"overlap": not args.no_overlap, "overlap_passes": args.overlap_passes,
             "overlap_sms": args.overlap_sms, "overlap_chunks": args.overlap_chunks, "tc_schedule": "dynamic" if args.dynamic_tiles else "static",
             "product_prefix": not args.no_prefix}
    st0 = rcs.State.build(ctx, circuit, fuse_k=args.fuse_k, amps=amps, keep_layout=keep, **bopts)   # sizes scratch
    scratch = st0.scratch
    st0.free()
    x_dev = torch.empty(shots, dtype=torch.int64, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def step(timing):
        st = rcs.State.build(ctx, circuit, fuse_k=args.fuse_k, timing=timing, amps=amps, scratch=scratch,
                             keep_layout=keep, **bopts)
        rep = rcs_sample_report()
        err = rcs_error()
        import ctypes as C
        check(L.rcs_sample(st._h, shots, SHOT_SEED, 0, C.c_void_p(x_dev.data_ptr()), C.byref(rep), C.byref(err)),
              err, "rcs_sample")
        xr = st.xeb(x_dev)
        return st, rep.sample_ms, xr

    for _ in range(args.warmup):
        st, _, _ = step(False)
        st.free()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    l0 = L.rcs_kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    reports, sample_ms, xebs, pass_ms = [], [], [], []
    for _ in range(args.steps):
        st, sms, xr = step(True)
        reports.append(st.report)
        sample_ms.append(sms)
        xebs.append(xr)
        pass_ms.extend(st.pass_times().tolist())
        st.free()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = L.rcs_kernel_launches() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    pass_bytes_rank = reports[0]["pass_bytes"]
    total_pass_bytes = pass_bytes_rank * world * args.steps
    value = total_pass_bytes / (ms_max / 1e3) / 1e9

    # ---- e2e through the public API with host buffers
    e2e_steps = args.steps if args.e2e_steps < 0 else args.e2e_steps
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    up_bytes = 0
    e2e_plan_ms = []
    for _ in range(e2e_steps):
        c2 = rcs.Circuit.from_qasm(text)                       # host QASM in
        st = rcs.State.build(ctx, c2, fuse_k=args.fuse_k, amps=amps, scratch=scratch, keep_layout=keep, **bopts)
        up_bytes = st.report["upload_bytes"]                   # plan operands copied by this build
        e2e_plan_ms.append(st.report["plan_ms"])
        xh = st.sample(shots, seed=SHOT_SEED)                  # bitstrings to host
        xr_h = st.xeb(xh)                                      # XEB from the host array
        st.free()
    torch.cuda.synchronize()
    w_ms = (time.perf_counter() - w0) * 1e3
    t = torch.tensor([w_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e_value = pass_bytes_rank * world * e2e_steps / (e2e_ms / 1e3) / 1e9 if e2e_steps else None

    # ---- roofline of the dominant kernel (fused gate pass)
    peak, peak_src = measured_peak_hbm()
    per_launch = 16.0 * (1 << (n - g))
    mean_pass_ms = statistics.mean(pass_ms)
    achieved = per_launch / (mean_pass_ms / 1e3) / 1e9
    gbs = sorted(per_launch / (p / 1e3) / 1e9 for p in pass_ms)
    R = reports[-1]
    step_ms = ms_max / args.steps
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            proj, sdesc, cores, spent = oracle_sample(args.config, cfg, shots, args.cpu_budget)
            cpu = {"value": total_pass_bytes / args.steps / proj / 1e9, "unit": "GB/s", "cores": cores,
                   "kind": "oracle", "sample": sdesc, "projected": True, "projected_step_s": proj,
                   "cpu_seconds_spent": spent, "host": host_info()}
        X = xebs[-1]
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "dtype_note": ("complex64 state; 6-qubit passes on tcgen05 kind::f16 with an fp16 hi/lo split "
                           "(hi = integer-valued, per-row/per-column power-of-two scales): exact integer main "
                           "term + rounded cross terms, fp32 TMEM accumulation, fp32 epilogue; fp64 block CDF, "
                           "search and XEB"),
            "data": "synthetic: seeded Sycamore-style circuit (rcs_workload, seed 1), shot seed 2512",
            "config": {"workload": desc, "n_qubits": n, "cycles": cfg["cycles"], "pattern": cfg["pattern"],
                       "shots": shots, "fuse_k": R["fuse_k"],
                       "parallelism": (f"state sharded over top {g} qubit(s), remaps = in-place NVLink peer swaps "
                                               "pipelined with the neighbouring passes") if world > 1 else "1 GPU",
                       "l2": "no flush: state (%d GiB per GPU) >> 126 MB L2" % ((8 << (n - g)) >> 30),
                       "sampler": ("kept layout (no final restore): every rank all-gathers the physical block "
                                   "sums and scans the logical-order CDF of the whole state (2^(n-6) doubles, "
                                   "replicated); north_star's per-rank partial CDF + scan of shard totals is the "
                                   "--canonical path. Same picks at N=1; at N>1 the scan association differs "
                                   "(G17 band)") if keep and world > 1 else
                                  ("canonical layout: per-rank block CDF + exclusive scan of shard totals"
                                   if world > 1 else "block CDF (b=6) + per-shot search")},
            "build_s": statistics.median(r["build_ms"] for r in reports) / 1e3,
            "shots_per_s": shots / (statistics.median(sample_ms) / 1e3),
            "shots_per_s_incl_blocksum": shots / ((statistics.median(sample_ms) + R["blocksum_ms"]) / 1e3),
            "xeb": X["F"], "xeb_sigma": X["sigma"], "fstar": X["fstar"], "norm": R["norm"],
            "n_passes": R["n_passes"], "n_prefix": R["n_prefix"], "prefix_ms": R["prefix_ms"],
            "n_remaps": R["n_remaps"], "n_swaps": R["n_swaps"],
            "layout_kept": R["layout_kept"],
            "pass_gbs": {"min": gbs[0], "median": gbs[len(gbs) // 2], "max": gbs[-1]},
            "pass_ms_total": R["pass_ms"], "remap_ms_total": R["remap_ms"], "swap_ms_total": R["swap_ms"],
            "blocksum_ms": R["blocksum_ms"], "n_tc_passes": R["n_tc_passes"],
            "remap": {"bytes_per_rank": R["remap_bytes"], "exposed_ms": R["remap_ms"],
                      "kernel_ms": R["remap_kernel_ms"],
                      "nvlink_gbs": (R["remap_bytes"] / (R["remap_kernel_ms"] / 1e3) / 1e9)
                      if R["remap_kernel_ms"] > 0 else None,
                      "peak_gbs": 900.0,
                      "frac": (R["remap_bytes"] / (R["remap_kernel_ms"] / 1e3) / 1e9 / 900.0)
                      if R["remap_kernel_ms"] > 0 else None,
                      "note": ("bytes this rank moves out per step / device time of the swap kernels "
                               "(co-running with pass chunks when pipelined) vs NVLink 5's 900 GB/s per "
                               "direction; exposed_ms = remap time not hidden behind pass chunks")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_nominal_8tbs": achieved / 8000.0,
                         "traffic": ncu_traffic(args.config, world),
                         "kernel": ("k_pass_tc + k_pass_tct (6-qubit tcgen05 passes)" if R["n_tc_passes"] == R["n_passes"]
                                    else "gate passes (k_pass_tc + k_pass_pair/k_pass_bit0)"),
                         "per_launch_bytes": per_launch,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GB/s", "steps": e2e_steps, "ms_per_step": e2e_ms / max(1, e2e_steps),
                    "h2d_bytes_per_step": up_bytes + 8 * shots, "d2h_bytes_per_step": 8 * shots + 8,
                    "xeb": xr_h["F"] if e2e_steps else None,
                    "plan_ms": statistics.median(e2e_plan_ms) if e2e_steps else None},
            "gpu_launches": launches,
            "clocks": clk,
        }
        emit(out)
        print(f"[bench] {desc}: build {out['build_s']:.3f} s, {R['n_passes']} passes, pass GB/s median "
              f"{out['pass_gbs']['median']:.0f} ({achieved / peak:.1%} of {peak:.0f}), shots/s {out['shots_per_s']:.3g}, "
              f"XEB {X['F']:.4f}+-{X['sigma']:.4f} (F* {X['fstar']:.4f})", file=sys.stderr)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cfg, shots, desc = workload(args)
    n = cfg["n_qubits"]
    world = args.gpus
    # the step's algorithmic bytes as the library counts them: 16 B per amplitude per executed pass
    # + 8 B per amplitude for the product-state prefix kernel (write only)
    npf = PLAN_PREFIX[args.config][args.fuse_k]
    step_bytes = ((PLAN_PASSES[args.config][args.fuse_k] - npf) * 16.0 + (8.0 if npf else 0.0)) * (1 << n)
    budget = max(2.0, min(args.cpu_budget, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(args.config, cfg, shots, budget)
    vals, spent = [], []
    sdesc, cores = "", 0
    for _ in range(args.steps):
        proj, sdesc, cores, sec = oracle_sample(args.config, cfg, shots, budget)
        vals.append(step_bytes / proj / 1e9)
        spent.append(sec)
    v = statistics.median(vals)
    out = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": statistics.median(spent) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeded circuit)",
           "config": {"workload": desc, "n_qubits": n, "shots": shots}, "impl": "reference",
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sdesc,
                            "projected": True, "host": host_info()},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)
    return out


_JSON_FD = None


def emit(out: dict) -> None:
    """The one JSON line, on the real stdout (everything else written to fd 1 goes to stderr)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(out) + "\n").encode())


def main():
    # keep stdout = one JSON line: libraries (NCCL's "NCCL version" banner at NCCL_DEBUG=VERSION,
    # which ignores NCCL_DEBUG_FILE) write to fd 1, so fd 1 becomes stderr and the line goes to a dup
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
