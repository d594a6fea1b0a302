#!/bin/bash
# 4-GPU box: benches only (N = 1 with the cpu baseline, 2, 4, 4 canonical layout).
TAG=${1:-b4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $OUT/bench_N1.json 2> $OUT/bench_N1.err
for M in 2 4; do
  DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
     --master-addr 127.0.0.1 --master-port 29546 bench.py --gpus $M --steps 3 --warmup 3 \
     > $OUT/bench_N$M.json 2> $OUT/bench_N$M.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29547 \
   bench.py --gpus 4 --steps 3 --warmup 3 --canonical > $OUT/bench_N4_canon.json 2> $OUT/bench_N4_canon.err
echo done > $OUT/done
