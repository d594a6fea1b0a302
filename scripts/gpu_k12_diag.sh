#!/bin/bash
# K12 diagnostic builds (wrong results, timing only) at ncu's base clock on C3: which resource
# paces a tile -- 1: one accumulator read per chunk, 2: no cross-term MMAs, 3: no stores.
cd "$(dirname "$0")/.."
O=gpurun_out/k12diag; mkdir -p $O
for V in ${DIAG_VARIANTS:-"base:" "oneacc:-DRCS_K12_DIAG=1" "nocross:-DRCS_K12_DIAG=2" "nostore:-DRCS_K12_DIAG=3"}; do
  tag=${V%%:*}; flags=${V#*:}
  RCS_NVCC_FLAGS="$flags" python -m paper_2512_07311_b200.build --force > $O/build_$tag.log 2>&1 || { echo "build $tag failed"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control base \
    --kernel-name-base demangled -k "regex:k_pass_tct" -s 30 -c 6 --csv --log-file $O/ncu_$tag.csv \
    python scripts/c3_build.py c3 > /dev/null 2>&1
  python - $O/ncu_$tag.csv "$tag" <<'PY'
import csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
h = rows[0]; d = {}
for r in rows[1:]:
    d.setdefault(r[h.index("ID")], {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
print(sys.argv[2], " ".join("%.2f(%.0f%%)" % (v["gpu__time_duration.sum"] / 1e6, v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in d.values()))
PY
done
python -m paper_2512_07311_b200.build --force > $O/build_default.log 2>&1
