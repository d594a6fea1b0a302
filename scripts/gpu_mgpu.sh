#!/bin/bash
# Multi-GPU check under gpurun --gpus N: parity tests (all modes) + bench at N (and N/2 when N=4)
# + the NVLink access-pattern microbenchmark.
TAG=${1:-mg}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 300 ./scripts/micro/p2p_bench $N 8 > $OUT/p2p_bench.txt 2>&1; [ $N -ge 4 ] && CUDA_VISIBLE_DEVICES=0,1 timeout 300 ./scripts/micro/p2p_bench 2 8 >> $OUT/p2p_bench.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > $OUT/mgpu_tests.log 2>&1; echo "rc=$?" >> $OUT/mgpu_tests.log
for M in $N $((N/2)); do
  [ $M -lt 2 ] && continue
  DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $M --steps 3 --warmup 3 \
      > $OUT/bench_c4_N$M.json 2> $OUT/bench_c4_N$M.err; echo "rc=$?" >> $OUT/bench_c4_N$M.err
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $M --steps 3 --warmup 3 --no-overlap \
      > $OUT/bench_c4_N${M}_seq.json 2> $OUT/bench_c4_N${M}_seq.err; echo "rc=$?" >> $OUT/bench_c4_N${M}_seq.err
done
echo done > $OUT/done
