#!/bin/bash
# TC iteration: correctness subset, c3/c4 bench, ncu --set full of one TC pass.
TAG=${1:-tci}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "all_k or baseline_configs or sampling_and_xeb or virtual_global" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT3 > $OUT/plain_c3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 3 -c 1 \
      -o $OUT/prof_tc_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
fi
echo done > $OUT/done
