#!/bin/bash
# multi-GPU check (gpurun --gpus 4): parity tests; C4 N = 1, 2 and 4; C5 N = 4 (defaults)
cd "$(dirname "$0")/.."
OUT=gpurun_out/${MOUT:-mgpu}; mkdir -p $OUT
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 2400 python -m pytest tests/test_multigpu.py tests/test_multigpu_fullscale.py -q -s -p no:cacheprovider > $OUT/mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed" $OUT/mgpu_tests.log | tail -20
for M in 2 4; do
  DEV=$(seq -s, 0 $((M-1)))
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $M \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $M --steps 5 --warmup 3 \
      > $OUT/bench_c4_N$M.json 2> $OUT/bench_c4_N$M.err; echo "bench N=$M rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_c4_N$M.json'));r=d['remap'];print('N=$M', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), 'exposed', round(r['exposed_ms'],1), 'nvlink', round(r['nvlink_gbs'] or 0), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench_c4_N1.json 2> $OUT/bench_c4_N1.err; echo "bench N=1 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c4_N1.json'));print('N=1', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus 4 --config c5 --steps 3 --warmup 3 > $OUT/bench_c5_N4.json 2> $OUT/bench_c5_N4.err; echo "bench c5 N=4 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c5_N4.json'));r=d['remap'];print('C5 N=4', round(d['ms_per_step'],1), round(d['value']), d['xeb'], d['xeb_sigma'], d['norm'], 'exposed', round(r['exposed_ms'],1))"
