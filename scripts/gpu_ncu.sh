#!/bin/bash
# ncu evidence (1 GPU): C4 launch list (serialized per-launch times), one --set full
# capture per tensor-core kernel variant on C3 (K9 with 2 low targets, K12 without and with a
# permuted t bit), DRAM bytes of the K12 pass at C4.  Each command first runs without ncu.
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu; mkdir -p $OUT
python -m paper_2512_07311_b200.build > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
SHORT4="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
SHORT3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 $SHORT4 > $OUT/plain_c4.json 2> $OUT/plain_c4.err; echo "plain c4 rc=$?"
timeout 600 $SHORT3 > $OUT/plain_c3.json 2> $OUT/plain_c3.err; echo "plain c3 rc=$?"
if [ -z "$NCU_SKIP_LIST" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_c4.csv $SHORT4 > $OUT/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k regex:k_pass_tct -s 2 -c 1 --csv --log-file $OUT/dram_c4_k12.csv $SHORT4 > $OUT/ncu_dram.log 2>&1; echo "dram rc=$?"
fi
for spec in "k9:regex:k_pass_tc<:0" "k12:regex:k_pass_tct<.int.-1>:0" "k12p0:regex:k_pass_tct<.int.0>:0"; do
  IFS=: read tag kind rx skip <<< "$spec"
  timeout 1800 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "$kind:$rx" -s $skip -c 1 \
      -o $OUT/full_c3_$tag -f $SHORT3 > $OUT/ncu_full_$tag.log 2>&1; echo "full $tag rc=$?"
  ncu -i $OUT/full_c3_$tag.ncu-rep --page raw --csv > $OUT/full_c3_${tag}_raw.csv 2>/dev/null
  ncu -i $OUT/full_c3_$tag.ncu-rep --page details --csv > $OUT/full_c3_${tag}_details.csv 2>/dev/null
done
ls -la $OUT
