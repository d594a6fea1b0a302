#!/bin/bash
TAG=${1:-rounds}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests/test_multigpu.py -q -x > $OUT/mgpu_tests.log 2>&1; echo "rc=$?" >> $OUT/mgpu_tests.log
run() {  # M rounds tag extra-env
  local M=$1 R=$2 T=$3; local DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV RCS_SWAP_ROUNDS=$R timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
     --master-addr 127.0.0.1 --master-port 29545 bench.py --gpus $M --steps 3 --warmup 3 --no-cpu-baseline $4 \
     > $OUT/b_N${M}_r${R}_$T.json 2> $OUT/b_N${M}_r${R}_$T.err
}
run 4 1 kept; run 4 0 kept; run 4 1 canon --canonical; run 4 0 canon --canonical; run 2 1 kept
RCS_OVERLAP=0 run 4 1 seq; RCS_OVERLAP=0 run 4 0 seq
echo done > $OUT/done
