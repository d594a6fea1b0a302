#!/bin/bash
# 1-GPU: TC-pass parity tests, bench c4/c3, ncu launch list + --set full capture of k_pass_tc.
TAG=${1:-tc3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT3 > $OUT/plain_c3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 5 -c 1 \
      -o $OUT/prof_tc_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
fi
echo done > $OUT/done
