#!/bin/bash
# 1-GPU check (gpurun): build, quick parity, C4 bench, per-pass report, full GPU suite, smoke, prefix A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2512_07311_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.log; exit 1; }
timeout 300 python - > gpurun_out/quick.log 2>&1 <<'PY'
import numpy as np, oracle, paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm, random_qasm
ctx = rcs.Context(0)
for name, t in (("c2", config_qasm("c2")), ("rand20", random_qasm(20, 400, 3)), ("rand17", random_qasm(17, 300, 4))):
    ref = oracle.build_state(t)
    for rep in range(2):
        for kern in ("auto", "k9"):
            st = rcs.State.build(ctx, rcs.Circuit.from_qasm(t), fuse_k=6, tc_kernel=kern)
            d = st.copy_out().astype(np.complex128) - ref
            print(name, kern, st.report["n_passes"], np.abs(d).max(), np.linalg.norm(d), st.norm - 1, flush=True)
PY
rc=$?; cat gpurun_out/quick.log; [ $rc -eq 0 ] || { echo QUICK FAILED rc=$rc; exit 1; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/check_bench.json'));print(d['ms_per_step'],d['value'],d['pass_gbs'],d['roofline']['frac'],d['clocks'],d['norm'])"
timeout 300 python scripts/pass_report.py c4 6 > gpurun_out/check_pass_report.txt 2>&1; tail -45 gpurun_out/check_pass_report.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check_gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/check_gputests.log | tail -30
timeout 300 python __graft_entry__.py smoke > gpurun_out/check_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/check_smoke.log
for rep in 1 2; do
  for V in "prefix:" "noprefix:--no-prefix"; do
    tag=${V%%:*}; flags=${V#*:}
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 $flags > gpurun_out/check_${tag}_$rep.json 2> gpurun_out/check_${tag}_$rep.err
    python -c "import json;d=json.load(open('gpurun_out/check_${tag}_$rep.json'));print('$tag $rep', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), d['n_passes'], d.get('n_prefix'), d['clocks']['sm_mhz'])"
  done
done
