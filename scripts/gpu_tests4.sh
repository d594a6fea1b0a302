#!/bin/bash
TAG=${1:-t4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
echo done > $OUT/done
