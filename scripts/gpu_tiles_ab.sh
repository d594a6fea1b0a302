#!/bin/bash
# round-2 GPU check: K12 dynamic tile scheduler vs static, A/B on one box (alternating)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02i
OUT=gpurun_out/r02i
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; cat $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu.py -q -p no:cacheprovider -k "dynamic or transposed or c2 or precision" > $OUT/quick_tests.log 2>&1; echo "quick tests rc=$?"; tail -2 $OUT/quick_tests.log
for rep in 1 2; do
  for V in "static:" "dyn:--dynamic-tiles"; do
    tag=${V%%:*}; flags=${V#*:}
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 $flags > $OUT/bench_${tag}_$rep.json 2> $OUT/bench_${tag}_$rep.err
    python -c "import json;d=json.load(open('$OUT/bench_${tag}_$rep.json'));print('$tag $rep', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"
  done
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $OUT/gputests.log | tail -20
