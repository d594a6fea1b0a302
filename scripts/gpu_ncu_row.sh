#!/bin/bash
# ncu --set full of K12's row variant (k_pass_tct<9>) and a plain K12 launch on C4 (after a plain run)
cd "$(dirname "$0")/.."
O=gpurun_out/ncu_row; mkdir -p $O
python -m paper_2512_07311_b200.build > /dev/null 2>&1
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 $SHORT4 > $O/plain.json 2>&1; echo "plain rc=$?"
for spec in ${NCU_SPECS:-"row:k_pass_tct<.int.9>" "plain:k_pass_tct<.int.-1>"}; do
  tag=${spec%%:*}; rx=${spec#*:}
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$rx" -c 1 \
      -o $O/full_$tag -f $SHORT4 > $O/ncu_$tag.log 2>&1; echo "full $tag rc=$?"
  ncu -i $O/full_$tag.ncu-rep --page details --csv > $O/full_${tag}_details.csv 2>/dev/null
  ncu -i $O/full_$tag.ncu-rep --page raw --csv > $O/full_${tag}_raw.csv 2>/dev/null
done
