#!/bin/bash
# sweep (gpurun --gpus 4) after the round-2 pass speedups: SMs left to the swaps x passes chained
# behind a remap x chunk bits, C4 at N = 4 and 2, one box
cd "$(dirname "$0")/.."
OUT=gpurun_out/sweep5; mkdir -p $OUT
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() {  # M tag flags...
  local M=$1 tag=$2; shift 2
  local DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $M --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" \
      > $OUT/N${M}_$tag.json 2> $OUT/N${M}_$tag.err
  python -c "import json;d=json.load(open('$OUT/N${M}_$tag.json'));r=d['remap'];print('N=$M $tag', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), 'exposed', round(r['exposed_ms'],1), 'nvlink', round(r['nvlink_gbs'] or 0), d['clocks']['sm_mhz'])"
}
run 4 default
for sms in 16 24; do for ch in 5 8; do run 4 s${sms}_c${ch} --overlap-sms $sms --overlap-passes $ch; done; done
run 4 s16_c5_k3 --overlap-sms 16 --overlap-passes 5 --overlap-chunks 3
run 2 default
for sms in 24 32; do run 2 s${sms}_c5 --overlap-sms $sms --overlap-passes 5; done
