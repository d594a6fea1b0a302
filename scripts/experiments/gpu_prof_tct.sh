#!/bin/bash
TAG=${1:-ptct}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT3 > $OUT/plain_c3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_tct -s 2 -c 1 \
      -o $OUT/prof_tct_c3 $SHORT3 > $OUT/ncu_tct.log 2>&1
  timeout 900 ncu --set full --clock-control base --import-source on -k regex:k_pass_tct -s 2 -c 1 \
      -o $OUT/prof_tct_c3_base $SHORT3 > $OUT/ncu_tct_base.log 2>&1
fi
echo done > $OUT/done
