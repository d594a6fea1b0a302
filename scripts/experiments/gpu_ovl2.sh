#!/bin/bash
# Sweep: SMs reserved for the pipelined swaps x swap vector depth, at N=2 and N=4.
TAG=${1:-ovl2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() {  # M sms tag
  local M=$1 S=$2 T=$3; local DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV RCS_OVERLAP_SMS=$S timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
     --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus $M --steps 3 --warmup 3 --no-cpu-baseline \
     > $OUT/b_N${M}_s${S}_$T.json 2> $OUT/b_N${M}_s${S}_$T.err
}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for M in 4 2; do run $M 16 u4; run $M 24 u4; run $M 32 u4; done
RCS_NVCC_FLAGS=-DRCS_SWAP_U=8 python -c "from paper_2512_07311_b200 import build; build.build(force=True)" >> $OUT/build.log 2>&1
for M in 4 2; do run $M 16 u8; run $M 24 u8; run $M 32 u8; done
python -c "from paper_2512_07311_b200 import build; build.build(force=True)" >> $OUT/build.log 2>&1
echo done > $OUT/done
