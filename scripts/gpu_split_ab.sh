#!/bin/bash
# live (power-capped) A/B on one box, alternating: K12 D split by output half vs one N = 128 group
cd "$(dirname "$0")/.."
O=gpurun_out/${AB_OUT:-split_ab}; mkdir -p $O
for rep in 1 2; do
  for V in ${AB_VARIANTS:-"split:" "nosplit:-DRCS_K12_NSPLIT=0"}; do
    tag=${V%%:*}; flags=${V#*:}
    RCS_NVCC_FLAGS="$flags" python -m paper_2512_07311_b200.build --force > $O/build_$tag.log 2>&1 || { echo "build $tag failed"; continue; }
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/${tag}_$rep.json 2> $O/${tag}_$rep.err
    python -c "import json;d=json.load(open('$O/${tag}_$rep.json'));print('$tag $rep', round(d['ms_per_step'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"
  done
done
python -m paper_2512_07311_b200.build --force > /dev/null 2>&1
