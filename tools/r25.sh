export PDG_DEBUG_M=2
for cfg in "X=0" "PDG_ND_STAGE_KB=12" "PDG_ND_STAGE_KB=16" "PDG_ND_PF=8" "PDG_ND_PF=24" "PDG_ND_CHUNKS=8" "PDG_ND_CHUNKS=24" "PDG_ND_FLOW_LEAF=96" "PDG_ND_FLOW_LEAF=192" "PDG_ND_LEAF=96" "PDG_ND_LEAF=192"; do echo "=== $cfg"; env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|rror" | sed 's/fronts.*vmax/vmax/'; done > gpurun_out/sweep4.log 2>&1
