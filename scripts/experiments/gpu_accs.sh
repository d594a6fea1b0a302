#!/bin/bash
# 1-GPU: full GPU tests (default build), then the accumulator-count experiment (3/2/1): precision
# (parity subset + C4 norm) and sustained speed/power.
TAG=${1:-acc}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
for A in 3 2 1; do
  RCS_NVCC_FLAGS="-DRCS_TC_ACCS=$A" python -c "from paper_2512_07311_b200 import build; build.build(force=True)" >> $OUT/build.log 2>&1
  timeout 600 python -m pytest tests/test_gpu.py -q -k "random_circuits_all_k or baseline_configs or full_size" > $OUT/parity_a$A.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4_a$A.json 2> $OUT/bench_c4_a$A.err
  timeout 120 python scripts/power_probe.py pass > $OUT/power_a$A.txt 2>&1
done
python -c "from paper_2512_07311_b200 import build; build.build(force=True)" >> $OUT/build.log 2>&1
echo done > $OUT/done
