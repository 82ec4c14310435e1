timeout 300 python tools/debug_nd.py 128 > gpurun_out/nd_debug.log 2>&1; echo "dbg rc $?"
for cfg in "PDG_ND_NODEP=1" "PDG_ND_NOMATH=1 PDG_ND_NODEP=1" "PDG_ND_LEAF=256" "PDG_ND_LEAF=64"; do
  echo "=== $cfg"
  env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve"
done > gpurun_out/nd_sweep.log 2>&1
