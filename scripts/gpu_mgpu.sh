#!/bin/bash
# Multi-GPU check under gpurun --gpus N: parity test + bench at N.
TAG=${1:-mg}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $OUT/mgpu_tests.log 2>&1; echo "rc=$?" >> $OUT/mgpu_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 3 --warmup 3 > $OUT/bench_c4_N$N.json 2> $OUT/bench_c4_N$N.err; echo "rc=$?" >> $OUT/bench_c4_N$N.err
echo done > $OUT/done
