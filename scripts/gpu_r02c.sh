#!/bin/bash
# round-2 GPU check #3: full-scale pins + edge sampling + smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2512_07311_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02c_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02c_smoke.log
timeout 1200 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu.py -k "fullscale or edge or separable or product or inverse" -q -s -p no:cacheprovider > gpurun_out/r02c_tests.log 2>&1; echo "pytest rc=$?"
grep -E "^(FAILED|ERROR)|passed|failed|n=34 separable" gpurun_out/r02c_tests.log | tail -30
