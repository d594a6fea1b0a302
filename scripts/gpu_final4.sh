#!/bin/bash
# 4-GPU box, end of round: GPU suite, smoke(), then the bench lines (N = 1, 2, 4, 4 canonical).
TAG=${1:-f4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1
bash scripts/gpu_bench4.sh $TAG/bench
echo done > $OUT/done
