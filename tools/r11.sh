for cfg in "PDG_ND_NODEP=1" "PDG_ND_NOMATH=1 PDG_ND_NODEP=1"; do
  echo "=== $cfg"
  env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep -v "^  backward\|repeat"
done > gpurun_out/nd_sweep.log 2>&1
