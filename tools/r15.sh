for cfg in "X=0" "PDG_ND_STAGE_KB=8" "PDG_ND_STAGE_KB=16" "PDG_ND_STAGE_KB=24" "PDG_ND_PF=4" "PDG_ND_PF=32" "PDG_ND_PF=64" "PDG_ND_CHUNKS=4" "PDG_ND_CHUNKS=8" "PDG_ND_CHUNKS=32" "PDG_ND_NODEP=1 PDG_ND_NOMATH=1" "PDG_ND_NOMATH=1" "PDG_ND_STAGES=4" "PDG_ND_LEAF=96" "PDG_ND_LEAF=192"; do
  echo "=== $cfg"
  env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|Error\|error" | sed 's/fronts.*total/total/'
done > gpurun_out/nd_sweep2.log 2>&1
