#!/bin/bash
TAG=${1:-pair3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 python scripts/experiments/pair_check.py c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "bitwise_equal True" $OUT/check_small.txt; then
  for cfg in "3 12" "2 16" "4 24"; do
    set -- $cfg
    RCS_PAIR_DEPTH=$1 RCS_PAIR_SLACK=$2 timeout 300 python scripts/experiments/pair_check.py c3 c4 > $OUT/check_d$1_s$2.txt 2>&1
  done
  SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc_multi -s 3 -c 1 \
      -o $OUT/prof_pair_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
fi
echo done > $OUT/done
