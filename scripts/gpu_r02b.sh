#!/bin/bash
# round-2 GPU check #2: race fix in the exact-main kernels; full GPU suite incl. n=34 pins; precision; C4 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2512_07311_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.log; exit 1; }
timeout 300 python - > gpurun_out/quick.log 2>&1 <<'PY'
import numpy as np, oracle, paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm
ctx = rcs.Context(0)
for cfg in ("c1", "c2"):
    t = config_qasm(cfg); ref = oracle.build_state(t)
    for rep in range(3):
        for kern in ("auto", "k9"):
            st = rcs.State.build(ctx, rcs.Circuit.from_qasm(t), fuse_k=6, tc_kernel=kern)
            d = st.copy_out().astype(np.complex128) - ref
            print(cfg, kern, st.report["n_passes"], np.abs(d).max(), np.linalg.norm(d), st.norm - 1, flush=True)
PY
rc=$?; cat gpurun_out/quick.log; [ $rc -eq 0 ] || { echo QUICK FAILED rc=$rc; exit 1; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
head -c 4000 gpurun_out/r02b_bench.json; tail -2 gpurun_out/r02b_bench.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/r02b_gputests.log | tail -30
timeout 600 python scripts/precision_probe.py --out gpurun_out/r02_precision.txt 2>&1 | tail -12
