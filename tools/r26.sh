export PDG_DEBUG_M=2
for cfg in "X=0" "PDG_ND_ARENA_KB=80" "PDG_ND_ARENA_KB=64" "PDG_ND_ARENA_KB=48" "PDG_ND_ARENA_KB=64 PDG_ND_NODEP=1" "PDG_ND_NODEP=1"; do echo "=== $cfg"; env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|rror" | sed 's/fronts.*vmax/vmax/'; done > gpurun_out/sweep5.log 2>&1
