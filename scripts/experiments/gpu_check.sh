#!/bin/bash
# One GPU-box round: tests, bench, launch list, one ncu --set full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "rc=$?" >> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "rc=$?" >> $OUT/bench_c3.err
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
SHORT4="python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT4 > $OUT/plain_c4.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches_c4.csv $SHORT4 > $OUT/ncu_launch_c4.log 2>&1
fi
if timeout 600 $SHORT3 > $OUT/plain_c3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 2 \
      -o $OUT/prof_pass_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
fi
echo done > $OUT/done
