#!/bin/bash
# 4 GPUs: the n=36 config (BJ configs[4], 512 GiB state) sharded over 4 B200 (128 GiB each).
TAG=${1:-c5}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 \
   bench.py --config c5 --gpus 4 --steps 3 --warmup 3 > $OUT/bench_c5_N4.json 2> $OUT/bench_c5_N4.err
nvidia-smi --query-gpu=memory.total --format=csv > $OUT/mem.txt
echo done > $OUT/done
