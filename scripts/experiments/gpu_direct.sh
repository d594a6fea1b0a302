#!/bin/bash
TAG=${1:-direct}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
if grep -q "rc=0" $OUT/tests.log; then
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
  RCS_TC_NODIRECT=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_nodirect.json 2> $OUT/bench_c4_nodirect.err
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_2.json 2> $OUT/bench_c4_2.err
  timeout 120 python scripts/pass_report.py c4 6 > $OUT/pass_c4.txt 2>&1
  SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 0 -c 12 \
      -o $OUT/prof_c3_12 $SHORT3 > $OUT/ncu.log 2>&1
fi
echo done > $OUT/done
