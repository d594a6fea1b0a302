#!/bin/bash
TAG=${1:-pair2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 python scripts/experiments/pair_check.py c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "bitwise_equal True" $OUT/check_small.txt; then
  for cfg in "3 12" "2 8" "4 16" "6 16" "3 24"; do
    set -- $cfg
    RCS_PAIR_DEPTH=$1 RCS_PAIR_SLACK=$2 timeout 300 python scripts/experiments/pair_check.py c3 c4 > $OUT/check_d$1_s$2.txt 2>&1
  done
fi
echo done > $OUT/done
