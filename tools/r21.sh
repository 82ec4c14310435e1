for cfg in "X=0" "PDG_ND_STAGE_KB=16" "PDG_ND_STAGE_KB=20" "PDG_ND_STAGE_KB=24" "PDG_ND_STAGES=8" "PDG_ND_PF=8" "PDG_ND_PF=32" "PDG_ND_CHUNKS=8" "PDG_ND_LEAF=96" "PDG_ND_LEAF=160"; do
  echo "=== $cfg"
  env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|Error\|error" | sed 's/fronts.*vmax/vmax/'
done > gpurun_out/nd_sweep3.log 2>&1
