#!/bin/bash
# 1-GPU check: quick K12/K9 parity vs the oracle, C4 bench, K12 per-launch time at ncu's base
# clock and unlocked (SM-cycle bound?), prefix-kernel time, whole GPU suite, smoke.
cd "$(dirname "$0")/.."
O=gpurun_out/${CHECK:-check4}; mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || { echo BUILD FAILED; cat $O/build.log; exit 1; }
timeout 300 python - > $O/quick.log 2>&1 <<'PY'
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
rc=$?; cat $O/quick.log; [ $rc -eq 0 ] || { echo QUICK FAILED rc=$rc; exit 1; }
timeout 900 python bench.py > $O/bench_c4_N1.json 2> $O/bench_c4_N1.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_c4_N1.json'));print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['n_passes'],d['prefix_ms'],d['blocksum_ms'],d['e2e']['ms_per_step'],d['e2e'].get('plan_ms'),d['pass_gbs'],d['clocks'])"
timeout 300 python scripts/pass_report.py c4 6 > $O/pass_report.txt 2>&1; tail -32 $O/pass_report.txt
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
for cc in base none; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control $cc --kernel-name-base demangled -k regex:"k_pass_tc|k_product" -c 12 --csv --log-file $O/c3_tc_clock_$cc.csv $SHORT3 > $O/ncu_c3_$cc.log 2>&1; echo "c3 $cc rc=$?"
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $O/gputests.log | tail -20
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
