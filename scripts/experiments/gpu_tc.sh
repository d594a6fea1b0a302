#!/bin/bash
TAG=${1:-tc}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "all_k and 6" > $OUT/tc_first.log 2>&1; echo "rc=$?" >> $OUT/tc_first.log
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 600 python bench.py --config c4 --no-cpu-baseline > $OUT/bench_c4_k6.json 2> $OUT/bench_c4_k6.err; echo "rc=$?" >> $OUT/bench_c4_k6.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3_k6.json 2> $OUT/bench_c3_k6.err; echo "rc=$?" >> $OUT/bench_c3_k6.err
echo done > $OUT/done
