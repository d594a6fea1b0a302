#!/bin/bash
# Final 1-GPU evidence (gpurun): C4 bench (full contract), per-pass report, ncu launch list of one
# step, DRAM bytes of a K12 C4 launch, whole GPU suite, smoke.  Each ncu command runs after the
# same command has exited 0 without ncu.
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || { echo BUILD FAILED; cat $O/build.log; exit 1; }
timeout 900 python bench.py > $O/bench_c4_N1.json 2> $O/bench_c4_N1.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_c4_N1.json'));print(d['ms_per_step'],d['value'],d['roofline'],d['prefix_ms'],d['blocksum_ms'],d['e2e'],d['clocks'])"
timeout 300 python scripts/pass_report.py c4 6 > $O/pass_report_c4.txt 2>&1; tail -3 $O/pass_report_c4.txt
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 $SHORT4 > $O/plain_c4.json 2> $O/plain_c4.err; echo "plain c4 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c4.csv $SHORT4 > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k regex:"k_pass_tct|k_product|k_block_sums" -c 4 --csv --log-file $O/dram_c4.csv $SHORT4 > $O/ncu_dram.log 2>&1; echo "dram rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $O/gputests.log | tail -20
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
