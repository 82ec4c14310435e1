for cfg in "X=0" "PDG_ND_TILE8=1" "X=1" "PDG_ND_NODEP=1" "PDG_ND_NODEP=1 PDG_ND_TILE8=1"; do echo "=== $cfg"; env $cfg timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve\|identical" | sed 's/fronts.*total/total/'; done > gpurun_out/g8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_g8.log 2>&1; echo "pytest rc $?"
timeout 600 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench_g8.json 2>/dev/null
