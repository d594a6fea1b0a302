#!/bin/bash
TAG=${1:-trans2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 90 python scripts/experiments/trans_check.py rand22 c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "rc=0" $OUT/check_small.txt; then
  timeout 300 python scripts/experiments/trans_check.py c3 c4 > $OUT/check_big.txt 2>&1; echo "rc=$?" >> $OUT/check_big.txt
  timeout 900 python -m pytest tests/test_gpu.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
  SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tct -s 2 -c 1 \
      -o $OUT/prof_tct_c3 $SHORT3 > $OUT/ncu_tct.log 2>&1
fi
echo done > $OUT/done
