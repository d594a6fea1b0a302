#!/bin/bash
TAG=${1:-pd}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python scripts/experiments/power_kinds_dense.py > $OUT/power_kinds_dense.txt 2>&1; echo "rc=$?" >> $OUT/power_kinds_dense.txt
echo done > $OUT/done
