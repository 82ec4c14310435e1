timeout 120 python tools/debug_nd.py 128 > gpurun_out/nd_debug2.log 2>&1; echo "dbg rc $?"
PDG_ND_NODEP=1 timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve" > gpurun_out/nd_nodep2.log; echo "nodep rc $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_nd2.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench_nd2.json 2> gpurun_out/bench_nd2.err; echo "bench rc $?"
