#!/bin/bash
# 1 GPU: pass time vs targets above the 2 MB page, per-pass report at C4, ncu launch list (K9 + K12).
TAG=${1:-pages}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python scripts/experiments/pages_check.py 34 > $OUT/pages_34.txt 2>&1; echo "rc=$?" >> $OUT/pages_34.txt
timeout 600 python scripts/pass_report.py c4 6 > $OUT/pass_report_c4.txt 2>&1; echo "rc=$?" >> $OUT/pass_report_c4.txt
cp gpurun_out/pass_report_c4_k6.json $OUT/ 2>/dev/null
SHORT="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if timeout 600 $SHORT > $OUT/plain_c4.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches_c4.csv $SHORT > $OUT/ncu_launches.log 2>&1
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_pass_tct -s 2 -c 1 --csv --log-file $OUT/dram_tct_c4.csv $SHORT > $OUT/ncu_dram.log 2>&1
fi
echo done > $OUT/done
