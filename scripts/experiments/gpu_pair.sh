#!/bin/bash
TAG=${1:-pair}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 python scripts/experiments/pair_check.py c1 c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "bitwise_equal True" $OUT/check_small.txt; then
  timeout 300 python scripts/experiments/pair_check.py c3 c4 > $OUT/check_big.txt 2>&1; echo "rc=$?" >> $OUT/check_big.txt
  timeout 600 python -m pytest tests/test_gpu.py -q -x -k "paired or keep or random_circuits_all_k or baseline" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
  RCS_TC_PAIR=0 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_nopair.json 2> $OUT/bench_c4_nopair.err
  timeout 120 python scripts/power_probe.py pass > $OUT/power.txt 2>&1
fi
echo done > $OUT/done
