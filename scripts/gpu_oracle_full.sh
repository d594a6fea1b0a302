#!/bin/bash
# Full-state oracle comparison (scripts/oracle_c4_full.py) on the GPU box: C2 (n=24) as a
# quick check, then the C4 circuit at N_QUBITS (34 needs >= 280 GiB host RAM; 33 fits a 196 GiB box).
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/oracle_full
mkdir -p $O
python -m paper_2512_07311_b200.build > $O/build.log 2>&1 || exit 9
(free -g; nproc; lscpu | head -20) > $O/host.txt
timeout 300 python scripts/oracle_c4_full.py --config c2 --out $O/c2 > $O/c2.out 2>&1; echo c2 rc=$?
timeout 3300 python scripts/oracle_c4_full.py --config c4 --n-qubits ${N_QUBITS:-33} --out $O/c4 > $O/c4.out 2>&1; echo c4 rc=$?
tail -n 5 $O/c4.out
