#!/bin/bash
TAG=${1:-pw}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
{
timeout 120 python scripts/power_probe.py copy
RCS_TC_EXPERIMENT=0 timeout 120 python scripts/power_probe.py pass
RCS_TC_EXPERIMENT=1 timeout 120 python scripts/power_probe.py pass
RCS_TC_EXPERIMENT=2 timeout 120 python scripts/power_probe.py pass
timeout 120 python scripts/power_probe.py copy
RCS_TC_EXPERIMENT=0 timeout 120 python scripts/power_probe.py pass
} > $OUT/power.txt 2>&1
echo done > $OUT/done
