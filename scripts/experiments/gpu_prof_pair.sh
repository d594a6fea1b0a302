#!/bin/bash
TAG=${1:-ppair}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT3 > $OUT/plain_c3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tc_multi -s 3 -c 1 \
      -o $OUT/prof_pair_c3 $SHORT3 > $OUT/ncu_full_c3.log 2>&1
fi
echo done > $OUT/done
