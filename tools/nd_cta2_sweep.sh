#!/bin/bash
# Chunk kernel with two smaller CTAs per SM (4 compute warps, 1 staging, 2 gather): rebuilds nd.o with the
# variant macros and times the config-1 inner solves; restores the default build at the end. Run on the GPU box.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
MK=paper_1801_04984_b200/csrc
OBJ=paper_1801_04984_b200/_lib/obj/nd.o
run() { echo "-- $*"; env "$@" timeout 300 python tools/nd_time.py 30 2>&1 | tail -1; }
echo "== default build"; run X=0
for V in "128 1 2 2" "128 2 4 2" "64 1 2 2"; do
  set -- $V
  rm -f $OBJ
  if ! make -s -C $MK EXTRA="-DPDG_ND_THREADS=$1 -DPDG_ND_PREP=$2 -DPDG_ND_GATHER=$3 -DPDG_ND_MINB=$4" > /tmp/mk.log 2>&1; then
    echo "variant $V build failed: $(grep -m1 error /tmp/mk.log)"; continue
  fi
  echo "== THREADS=$1 PREP=$2 GATHER=$3 MINB=$4"
  run PDG_ND_STAGE_KB=12
  run PDG_ND_STAGE_KB=12 PDG_ND_LOCAL_DEPTH=7 PDG_ND_SPLIT_LOCAL=1
  run PDG_ND_STAGE_KB=8 PDG_ND_LOCAL_DEPTH=7 PDG_ND_SPLIT_LOCAL=1
  run PDG_ND_STAGE_KB=12 PDG_ND_LOCAL_DEPTH=7 PDG_ND_SPLIT_LOCAL=1 PDG_ND_HYBRID=1
  timeout 300 python -m pytest tests -m gpu -x -q -k "precond or inner" 2>&1 | tail -1
done
rm -f $OBJ; make -s -C $MK
