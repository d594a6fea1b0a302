#!/bin/bash
TAG=${1:-trans}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 90 python scripts/experiments/trans_check.py rand22 c2 > $OUT/check_small.txt 2>&1; echo "rc=$?" >> $OUT/check_small.txt
if grep -q "rc=0" $OUT/check_small.txt; then
  timeout 300 python scripts/experiments/trans_check.py c3 c4 > $OUT/check_big.txt 2>&1; echo "rc=$?" >> $OUT/check_big.txt
  timeout 900 python -m pytest tests/test_gpu.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
  RCS_TC_NOTRANS=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_k9.json 2> $OUT/bench_c4_k9.err
fi
echo done > $OUT/done
