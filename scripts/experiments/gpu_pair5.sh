#!/bin/bash
TAG=${1:-pair5}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
RCS_TC_PAIR=0 RCS_TC_MULTI1=1 timeout 300 python scripts/experiments/pair_check.py c2 c3 c4 > $OUT/check_multi1.txt 2>&1
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
RCS_PAIR_DEPTH=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc_multi -s 3 -c 1 \
      -o $OUT/prof_pair_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
echo done > $OUT/done
