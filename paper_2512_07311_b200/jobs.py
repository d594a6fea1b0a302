"""Paper stages 2-4 as independent jobs: snapshot -> N sampler jobs -> XEB.

PAPER §3.2 (l.36-39): one GPU builds the state, which "is written to a shared file system";
"N CPU-only jobs, each of which rebuilds the quantum state from the persisted state and
performs 2.5x10^6/N measurement shots ... Each job stores its output in a job-specific file";
post-processing "calculates the linear cross-entropy benchmarking (XEB) score".  Here a job is
an independent process that loads the snapshot onto a GPU (rcs_snapshot_load), draws its
shard with its own seed (rcs_job_seed), looks up p(x) for its distinct bitstrings
(rcs_probabilities) and writes result_<job_id>.jsonl (SPEC sampling-worker S:219-285):
    line 1: {"schema_version": 1, "job_id", "seed", "n_qubits", "shots", "snapshot_digest",
             "timings": {"queue_s", "load_s", "sample_s", "total_s"}}
    then one line per distinct bitstring: {"bitstring": "<n chars, qubit n-1 first>",
             "count": c, "p_ideal": p}
Every step of the arithmetic (load, digest, sampling, probabilities, XEB) runs in the library;
this module does process fan-out and file plumbing only.

    python -m paper_2512_07311_b200.jobs worker --snapshot s.rcss --shots 25000 --job-id 7 --out d
    python -m paper_2512_07311_b200.jobs pipeline --config c1 --shots 10000 --jobs 4 --work-dir d
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

SCHEMA = 1


def run_worker(snapshot: str, shots: int, base_seed: int, job_id: int, out_dir: str, queue_s: float = 0.0,
               device: int = 0) -> dict:
    """One stage-3 job; returns the header record (also written to result_<job_id>.jsonl)."""
    from . import Context, State, job_seed, snapshot_info
    t0 = time.perf_counter()
    if shots < 1:
        raise ValueError("shots must be >= 1")
    path = os.path.join(out_dir, f"result_{job_id}.jsonl")
    if os.path.exists(path):
        raise FileExistsError(path)      # jobs never overwrite
    ctx = Context(device)
    info = snapshot_info(snapshot)
    n = info["n_qubits"]
    t1 = time.perf_counter()
    st = State.load_snapshot(ctx, snapshot)
    t2 = time.perf_counter()
    seed = job_seed(base_seed, job_id)
    x = st.sample(shots, seed=seed)
    t3 = time.perf_counter()
    ux, counts = np.unique(x, return_counts=True)
    p = st.probabilities(ux)
    t4 = time.perf_counter()
    head = {"schema_version": SCHEMA, "job_id": job_id, "seed": seed, "n_qubits": n, "shots": int(shots),
            "snapshot_digest": info["digest"].hex(),
            "timings": {"queue_s": float(queue_s), "load_s": t2 - t1, "sample_s": t4 - t2,
                        "total_s": t4 - t0}}
    tmp = path + f".tmp.{os.getpid()}"
    with open(tmp, "w") as f:
        f.write(json.dumps(head) + "\n")
        for xi, ci, pi in zip(ux.tolist(), counts.tolist(), p.tolist()):
            f.write(json.dumps({"bitstring": format(int(xi), f"0{n}b"), "count": int(ci), "p_ideal": pi}) + "\n")
    try:
        os.link(tmp, path)               # atomic create-if-absent
    finally:
        os.unlink(tmp)
    st.free()
    return head


def read_result(path: str) -> tuple:
    """(header, x array, counts array, p array) of one result file."""
    with open(path) as f:
        head = json.loads(f.readline())
        xs, cs, ps = [], [], []
        for ln in f:
            r = json.loads(ln)
            xs.append(int(r["bitstring"], 2))
            cs.append(r["count"])
            ps.append(r["p_ideal"])
    return head, np.array(xs, np.uint64), np.array(cs, np.int64), np.array(ps, np.float64)


def aggregate(paths: list) -> dict:
    """Stage 4: XEB over all jobs' shots (each distinct bitstring weighted by its count)."""
    from . import xeb_from_probs
    heads, ps = [], []
    n = None
    for pth in paths:
        h, _, c, p = read_result(pth)
        heads.append(h)
        n = h["n_qubits"] if n is None else n
        if h["n_qubits"] != n or sum(c.tolist()) != h["shots"]:
            raise ValueError(f"inconsistent result file {pth}")
        ps.append(np.repeat(p, c))
    rep = xeb_from_probs(n, np.concatenate(ps))
    return {"n_qubits": n, "jobs": len(paths), "shots": int(rep["shots"]), "F": rep["F"], "sigma": rep["sigma"],
            "mean_p": rep["mean_p"], "job_timings": [h["timings"] for h in heads]}


def run_pipeline(qasm: str, total_shots: int, n_jobs: int, base_seed: int, work_dir: str, fuse_k: int = 0,
                 parallel: int = 1, device: int = 0) -> dict:
    """Stages 1-4 locally: build on `device`, snapshot, fan out n_jobs worker processes
    (`parallel` at a time, each on `device`), aggregate the result files."""
    from . import Circuit, Context, State, shard_shots
    if n_jobs < 1 or total_shots < n_jobs:
        raise ValueError(f"need 1 <= n_jobs <= total_shots (got n_jobs={n_jobs}, total_shots={total_shots}): "
                         "every job draws at least one shot")
    os.makedirs(work_dir, exist_ok=True)
    t0 = time.perf_counter()
    ctx = Context(device)
    st = State.build(ctx, Circuit.from_qasm(qasm), fuse_k=fuse_k)
    snap = os.path.join(work_dir, "state.rcss")
    digest = st.save_snapshot(snap)
    st.free()
    del ctx
    t1 = time.perf_counter()
    shards = shard_shots(total_shots, n_jobs)
    procs, paths, pending = [], [], list(enumerate(shards))
    env = dict(os.environ)
    try:
        while pending or procs:
            while pending and len(procs) < max(1, parallel):
                j, sh = pending.pop(0)
                cmd = [sys.executable, "-m", "paper_2512_07311_b200.jobs", "worker", "--snapshot", snap, "--shots",
                       str(sh), "--seed", str(base_seed), "--job-id", str(j), "--out", work_dir, "--device",
                       str(device), "--queue-s", f"{time.perf_counter() - t1:.6f}"]
                procs.append((j, subprocess.Popen(cmd, env=env)))
                paths.append(os.path.join(work_dir, f"result_{j}.jsonl"))
            for j, pr in list(procs):
                if pr.poll() is not None:
                    if pr.returncode != 0:
                        raise RuntimeError(f"job {j} failed with exit code {pr.returncode}")
                    procs.remove((j, pr))
            time.sleep(0.02)
    except BaseException:
        for _, pr in procs:   # no orphaned GPU workers: stop and reap the jobs still running
            if pr.poll() is None:
                pr.terminate()
        for _, pr in procs:
            try:
                pr.wait(timeout=30)
            except subprocess.TimeoutExpired:
                pr.kill()
                pr.wait()
        raise
    t2 = time.perf_counter()
    out = aggregate(paths)
    out.update({"snapshot": snap, "snapshot_digest": digest.hex(), "stage1_s": t1 - t0, "stage3_s": t2 - t1})
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2512_07311_b200.jobs")
    sub = ap.add_subparsers(dest="cmd", required=True)
    w = sub.add_parser("worker")
    w.add_argument("--snapshot", required=True)
    w.add_argument("--shots", type=int, required=True)
    w.add_argument("--seed", type=int, default=2512)
    w.add_argument("--job-id", type=int, default=None)
    w.add_argument("--out", required=True)
    w.add_argument("--device", type=int, default=0)
    w.add_argument("--queue-s", type=float, default=0.0)
    p = sub.add_parser("pipeline")
    p.add_argument("--qasm", default=None)
    p.add_argument("--config", default="c1")
    p.add_argument("--shots", type=int, default=None)
    p.add_argument("--jobs", type=int, default=4)
    p.add_argument("--seed", type=int, default=2512)
    p.add_argument("--work-dir", required=True)
    p.add_argument("--parallel", type=int, default=1)
    a = ap.parse_args(argv)
    if a.cmd == "worker":
        jid = a.job_id if a.job_id is not None else int(os.environ.get("SLURM_JOB_ID", "0"))
        run_worker(a.snapshot, a.shots, a.seed, jid, a.out, a.queue_s, a.device)
    else:
        if a.qasm:
            text = open(a.qasm).read()
            shots = a.shots or 10000
        else:
            from rcs_workload import CONFIGS, config_qasm
            text = config_qasm(a.config)
            shots = a.shots or CONFIGS[a.config]["shots"]
        print(json.dumps(run_pipeline(text, shots, a.jobs, a.seed, a.work_dir, parallel=a.parallel)))


if __name__ == "__main__":
    main()
