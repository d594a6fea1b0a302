#!/bin/bash
# round-2 multi-GPU check #2 (gpurun --gpus 4): pipelined remap chains (up to 3 passes behind a
# remap) vs the next pass only vs sequential; multi-GPU parity tests; C5 at N = 4
cd "$(dirname "$0")/.."
OUT=gpurun_out/mgpu2; mkdir -p $OUT
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > $OUT/mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $OUT/mgpu_tests.log | tail -20
for M in 2 4; do
  DEV=$(seq -s, 0 $((M-1)))
  for V in "chain:" "next:--overlap-passes 1" "seq:--no-overlap"; do
    tag=${V%%:*}; flags=${V#*:}
    CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
        --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $M --steps 5 --warmup 3 $flags \
        > $OUT/bench_c4_N${M}_$tag.json 2> $OUT/bench_c4_N${M}_$tag.err; echo "bench N=$M $tag rc=$?"
    python -c "import json;d=json.load(open('$OUT/bench_c4_N${M}_$tag.json'));r=d['remap'];print('N=$M $tag', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), 'exposed', round(r['exposed_ms'],1), 'nvlink', round(r['nvlink_gbs'] or 0), d['clocks']['sm_mhz'])"
  done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus 4 --config c5 --steps 3 --warmup 3 > $OUT/bench_c5_N4.json 2> $OUT/bench_c5_N4.err; echo "bench c5 N=4 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c5_N4.json'));r=d['remap'];print('C5 N=4', round(d['ms_per_step'],1), round(d['value']), d['xeb'], d['norm'], 'exposed', round(r['exposed_ms'],1))"
