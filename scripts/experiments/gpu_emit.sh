#!/bin/bash
# 2 GPUs: bench stdout is exactly one JSON line (N=1, N=2, reference arm at N=2).
TAG=${1:-emit}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $OUT/bench_N1.json 2> $OUT/bench_N1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29546 \
   bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_N2.json 2> $OUT/bench_N2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29547 \
   bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/ref_N2.json 2> $OUT/ref_N2.err
wc -l $OUT/*.json > $OUT/lines.txt
echo done > $OUT/done
