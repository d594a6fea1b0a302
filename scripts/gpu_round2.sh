#!/bin/bash
# Single-GPU round check: build, smoke, all GPU tests, benches, ncu launch list + TC-pass DRAM bytes at C4.
TAG=${1:-rr}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
SHORT="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT > $OUT/plain_c4.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches_c4.csv $SHORT > $OUT/ncu_launches.log 2>&1
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_pass_tc -s 3 -c 1 --csv --log-file $OUT/dram_c4.csv $SHORT > $OUT/ncu_dram.log 2>&1
fi
echo done > $OUT/done
