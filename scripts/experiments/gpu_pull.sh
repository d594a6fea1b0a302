#!/bin/bash
# 4-GPU box: multi-GPU tests, then C4 benches at N=4 (pull / swap) and N=2.
TAG=${1:-pull}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests/test_multigpu.py -q -x > $OUT/mgpu_tests.log 2>&1; echo "rc=$?" >> $OUT/mgpu_tests.log
run() {  # M pull tag
  local M=$1 P=$2; local DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV RCS_REMAP_PULL=$P timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
     --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $M --steps 3 --warmup 3 \
     > $OUT/b_N${M}_pull$P.json 2> $OUT/b_N${M}_pull$P.err
}
run 4 1; run 4 0; run 2 1
echo done > $OUT/done
