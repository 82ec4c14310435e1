set -x
timeout 300 python tools/debug_nd.py 128 > gpurun_out/nd_debug.log 2>&1; echo "dbg rc $?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 600 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
