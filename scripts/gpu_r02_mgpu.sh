#!/bin/bash
# round-2 multi-GPU check (gpurun --gpus 4): multi-GPU parity tests (world 2 and 4, all remap
# modes), C4 bench at N = 2 and 4 (pipelined and sequential remaps), C5 (n=36) at N = 4
cd "$(dirname "$0")/.."
OUT=gpurun_out/mgpu; mkdir -p $OUT
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > $OUT/mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $OUT/mgpu_tests.log | tail -20
for M in 2 4; do
  DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $M --steps 5 --warmup 3 \
      > $OUT/bench_c4_N$M.json 2> $OUT/bench_c4_N$M.err; echo "bench N=$M rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_c4_N$M.json'));print('N=$M', round(d['ms_per_step'],1), round(d['value']), d['roofline']['frac'], d['remap'], d['clocks'])"
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $M --steps 5 --warmup 3 --no-overlap \
      > $OUT/bench_c4_N${M}_seq.json 2> $OUT/bench_c4_N${M}_seq.err; echo "bench N=$M seq rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_c4_N${M}_seq.json'));print('N=$M seq', round(d['ms_per_step'],1), round(d['value']), d['remap'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus 4 --config c5 --steps 3 --warmup 3 > $OUT/bench_c5_N4.json 2> $OUT/bench_c5_N4.err; echo "bench c5 N=4 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c5_N4.json'));print('C5 N=4', round(d['ms_per_step'],1), round(d['value']), d['xeb'], d['norm'], d['remap'])"
