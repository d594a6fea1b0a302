#!/bin/bash
# Multi-GPU sweep of the pipelined-remap knobs (SMs left to the swaps, chunk count) at N=2 and N=4.
TAG=${1:-ovl}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() {   # M sms cb
  local M=$1 S=$2 CB=$3; local DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV RCS_OVERLAP_SMS=$S RCS_OVERLAP_CHUNKS=$CB timeout 600 python -m torch.distributed.run \
     --nnodes=1 --nproc-per-node $M --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus $M --steps 3 --warmup 3 \
     --no-cpu-baseline > $OUT/b_N${M}_s${S}_c${CB}.json 2> $OUT/b_N${M}_s${S}_c${CB}.err
}
for M in 2 4; do run $M 32 2; run $M 48 2; run $M 32 3; run $M 64 2; done
echo done > $OUT/done
