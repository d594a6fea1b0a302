#!/bin/bash
# ncu --set full of one C4 block-sum launch and one prefix launch (after a plain run)
cd "$(dirname "$0")/.."
O=gpurun_out/ncu_bsum; mkdir -p $O
python -m paper_2512_07311_b200.build > /dev/null 2>&1
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 $SHORT4 > $O/plain.json 2>&1; echo "plain rc=$?"
for k in k_block_sums k_product_init; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$k -c 1 \
      -o $O/full_$k -f $SHORT4 > $O/ncu_$k.log 2>&1; echo "full $k rc=$?"
  ncu -i $O/full_$k.ncu-rep --page details --csv > $O/full_${k}_details.csv 2>/dev/null
  ncu -i $O/full_$k.ncu-rep --page raw --csv > $O/full_${k}_raw.csv 2>/dev/null
done
