for cfg in "X=0" "PDG_ND_FENCE=1" "X=1" "PDG_ND_FENCE=1"; do echo "=== $cfg"; env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|identical" | sed 's/fronts.*total/total/'; done > gpurun_out/fence.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_fence.log 2>&1; echo "pytest rc $?"
