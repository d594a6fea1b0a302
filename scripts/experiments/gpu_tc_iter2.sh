#!/bin/bash
# TC iteration v2: correctness subset, per-pass report, c3/c4 bench.
TAG=${1:-tci}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "all_k or baseline_configs or sampling_and_xeb or virtual_global or full_size" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
timeout 300 python scripts/pass_report.py c3 6 > $OUT/pass_c3.txt 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
echo done > $OUT/done
