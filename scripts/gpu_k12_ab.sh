#!/bin/bash
# K12 build variants (D split by output half, pipelined epilogue) x TMA request shape, timed per
# launch by ncu at the base clock on C3 (cycle counts independent of the power cap), then the
# default build's full check.
cd "$(dirname "$0")/.."
O=gpurun_out/k12ab; mkdir -p $O
for V in "split+pipe:" "nosplit+pipe:-DRCS_K12_NSPLIT=0" "split+simple:-DRCS_K12_EPIPIPE=0" "nosplit+simple:-DRCS_K12_NSPLIT=0 -DRCS_K12_EPIPIPE=0"; do
  tag=${V%%:*}; flags=${V#*:}
  RCS_NVCC_FLAGS="$flags" python -m paper_2512_07311_b200.build --force > $O/build_$tag.log 2>&1 || { echo "build $tag failed"; continue; }
  for tma in auto bulk; do
    timeout 300 python scripts/c3_build.py c3 --tma $tma > $O/plain_${tag}_$tma.txt 2>&1 || { echo "run $tag $tma failed"; tail -3 $O/plain_${tag}_$tma.txt; continue; }
    timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control base \
      --kernel-name-base demangled -k regex:k_pass_tc -s 33 -c 12 --csv --log-file $O/ncu_${tag}_$tma.csv \
      python scripts/c3_build.py c3 --tma $tma > /dev/null 2>&1
    python - $O/ncu_${tag}_$tma.csv "$tag $tma" <<'PY'
import csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
h = rows[0]; d = {}
for r in rows[1:]:
    d.setdefault(r[h.index("ID")], {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
    d[r[h.index("ID")]]["k"] = r[h.index("Kernel Name")][:26]
print(sys.argv[2], " ".join("%s:%.2f" % (v["k"][-3:], v["gpu__time_duration.sum"] / 1e6) for v in d.values()))
PY
  done
done
python -m paper_2512_07311_b200.build --force > $O/build_default.log 2>&1
CHECK=k12ab/check bash scripts/gpu_check4.sh
