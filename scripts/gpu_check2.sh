#!/bin/bash
# 1-GPU check after the product-prefix row kernel + planner caches: prefix parity, C4 bench
# (full contract), per-pass clock/power trace, ncu launch list + the prefix kernel's DRAM bytes,
# then the whole GPU suite and smoke.
cd "$(dirname "$0")/.."
O=gpurun_out/check2; mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || { echo BUILD FAILED; cat $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu.py -q -p no:cacheprovider -k "product_prefix" > $O/prefix_tests.log 2>&1; echo "prefix tests rc=$?"; tail -2 $O/prefix_tests.log
timeout 900 python bench.py > $O/bench_c4_N1.json 2> $O/bench_c4_N1.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_c4_N1.json'));print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['prefix_ms'],d['e2e']['ms_per_step'],d['e2e'].get('plan_ms'),d['clocks'])"
timeout 600 python scripts/pass_power_trace.py --out $O/pass_power_c4.txt > $O/pass_power.log 2>&1; echo "trace rc=$?"; tail -3 $O/pass_power_c4.txt
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c4.csv $SHORT4 > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k regex:k_product -c 2 --csv --log-file $O/dram_c4_prefix.csv $SHORT4 > $O/ncu_dram.log 2>&1; echo "dram rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $O/gputests.log | tail -20
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
