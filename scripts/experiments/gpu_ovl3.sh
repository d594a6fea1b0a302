#!/bin/bash
# 4 GPUs: reserved-SM / chunk sweep of the pipelined remaps with the K12 code (N = 4 and N = 2).
TAG=${1:-ovl3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
for cfg in "4 8 2" "4 16 2" "4 24 2" "4 16 3" "4 24 3" "4 32 3" "2 24 2" "2 32 2" "2 48 2" "2 32 3"; do
  set -- $cfg; N=$1; S=$2; C=$3
  DEV=$(seq -s, 0 $((N-1)))
  CUDA_VISIBLE_DEVICES=$DEV RCS_OVERLAP_SMS=$S RCS_OVERLAP_CHUNKS=$C timeout 300 python -m torch.distributed.run \
     --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29550 $B --gpus $N \
     > $OUT/b_N${N}_s${S}_c${C}.json 2> $OUT/b_N${N}_s${S}_c${C}.err
done
echo done > $OUT/done
