#!/bin/bash
# 1-GPU A/B of the TC epilogue width: 8 warps (default) vs 4 warps.
TAG=${1:-tc4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_e8.json 2> $OUT/bench_c4_e8.err
timeout 120 python scripts/power_probe.py pass > $OUT/power_e8.txt 2>&1
RCS_NVCC_FLAGS=-DRCS_TC_EPI_WARPS=4 python -c "from paper_2512_07311_b200 import build; build.build(force=True)" >> $OUT/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_e4.json 2> $OUT/bench_c4_e4.err
timeout 120 python scripts/power_probe.py pass > $OUT/power_e4.txt 2>&1
echo done > $OUT/done
