#!/bin/bash
# Rebuilds the library with ND-kernel variants (compute threads, pipeline slots) and times
# config 1 with each; restores the default build at the end. Run on the GPU box.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
MK=paper_1801_04984_b200/csrc/Makefile
OBJ=paper_1801_04984_b200/_lib/obj/nd.o
for V in "256 8" "128 8" "384 8" "512 8" "256 4" "256 6"; do
  set -- $V
  rm -f $OBJ
  if ! make -s -f $MK EXTRA="-DPDG_ND_THREADS=$1 -DPDG_ND_BUFS=$2" > /tmp/mk.log 2>&1; then
    echo "ND_THREADS $1 BUFS $2 build failed: $(grep -m1 error /tmp/mk.log)"; continue
  fi
  timeout 120 python bench.py --steps 10 --warmup 3 --spmv-sizes 256 --spmv-reps 5 --no-cpu-baseline 2>/tmp/b.err \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ND_THREADS', $1, 'BUFS', $2, d['value'], d['iterations'][:3], d['phases']['a_solve']['ms_per_step'], d['phases']['flow_solve']['ms_per_step'])" \
    || echo "ND_THREADS $1 BUFS $2 run failed: $(tail -1 /tmp/b.err)"
done
rm -f $OBJ; make -s -f $MK
