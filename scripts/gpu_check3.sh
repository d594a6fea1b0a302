#!/bin/bash
# 1-GPU re-entry check (gpurun): C4 bench (full contract), whole GPU suite, smoke, C4 launch
# list, prefix-kernel DRAM bytes, and K12 at ncu's base clock (SM-side limit under the power cap).
cd "$(dirname "$0")/.."
O=gpurun_out/check3; mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || { echo BUILD FAILED; cat $O/build.log; exit 1; }
timeout 900 python bench.py > $O/bench_c4_N1.json 2> $O/bench_c4_N1.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_c4_N1.json'));print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['prefix_ms'],d['blocksum_ms'],d['e2e']['ms_per_step'],d['e2e'].get('plan_ms'),d['clocks'])"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $O/gputests.log | tail -20
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c4.csv $SHORT4 > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k regex:k_product -c 1 --csv --log-file $O/dram_c4_prefix.csv $SHORT4 > $O/ncu_dram.log 2>&1; echo "dram rc=$?"
for cc in base none; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control $cc --kernel-name-base demangled -k regex:k_pass_tc -c 12 --csv --log-file $O/c3_tc_clock_$cc.csv $SHORT3 > $O/ncu_c3_$cc.log 2>&1; echo "c3 $cc rc=$?"
done
