# ND inner-solve variants on config 1 (tools/nd_time.py); usage: bash tools/nd_sweep.sh "CFG1" "CFG2" ...
for cfg in "$@"; do
  printf "%-70s " "$cfg"
  env $cfg timeout 180 python tools/nd_time.py 30 2>&1 | tail -1
done
