#!/bin/bash
TAG=${1:-pair4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 python scripts/experiments/pair_check.py c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "bitwise_equal True" $OUT/check_small.txt; then
  for cfg in "2 16 18" "3 16 18" "2 16 19" "2 8 17"; do
    set -- $cfg
    RCS_PAIR_DEPTH=$1 RCS_PAIR_SLACK=$2 RCS_PAIR_MAXBITS=$3 timeout 300 python scripts/experiments/pair_check.py c3 c4 > $OUT/check_d$1_s$2_m$3.txt 2>&1
  done
fi
echo done > $OUT/done
