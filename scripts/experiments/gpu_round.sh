#!/bin/bash
# Full single-GPU round: all GPU tests, per-pass report, benches (c4 default incl. cpu baseline, c3).
TAG=${1:-rr}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 300 python scripts/pass_report.py c4 6 > $OUT/pass_c4.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
echo done > $OUT/done
