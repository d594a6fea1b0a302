#!/bin/bash
# 1-GPU: whole GPU suite + smoke, then ncu --set full (base clock) of the two K12 launch kinds on
# C3: r = 7 (64 TMA runs of 1 KB per tile) and r = 8 (32 runs of 2 KB).
cd "$(dirname "$0")/.."
O=gpurun_out/check5; mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || { echo BUILD FAILED; cat $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $O/gputests.log | tail -20
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
for spec in "k12r7:0" "k12r8:1"; do
  IFS=: read tag skip <<< "$spec"
  timeout 1200 ncu --set full --import-source on --clock-control base --kernel-name-base demangled -k "regex:k_pass_tct<.int.-1>" -s $skip -c 1 \
      -o $O/full_c3_$tag -f $SHORT3 > $O/ncu_full_$tag.log 2>&1; echo "full $tag rc=$?"
  ncu -i $O/full_c3_$tag.ncu-rep --page raw --csv > $O/full_c3_${tag}_raw.csv 2>/dev/null
  ncu -i $O/full_c3_$tag.ncu-rep --page details --csv > $O/full_c3_${tag}_details.csv 2>/dev/null
  ncu -i $O/full_c3_$tag.ncu-rep --page source --csv --print-source sass > $O/full_c3_${tag}_sass.csv 2>/dev/null
done
ls -la $O
