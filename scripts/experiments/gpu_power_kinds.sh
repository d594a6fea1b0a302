#!/bin/bash
TAG=${1:-pk}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/power_probe.py copy > $OUT/power_kinds.txt 2>&1
timeout 900 python scripts/experiments/power_kinds.py >> $OUT/power_kinds.txt 2>&1; echo "rc=$?" >> $OUT/power_kinds.txt
echo done > $OUT/done
