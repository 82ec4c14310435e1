for cfg in "PDG_ND_WARP_LD=0" "PDG_ND_WARP_LD=0 PDG_ND_STAGE_KB=12" ; do
  echo "=== $cfg"
  env $cfg timeout 300 python tools/debug_nd.py 128 2>&1 | grep -A25 "nd solve"
done > gpurun_out/nd_sweep.log 2>&1
