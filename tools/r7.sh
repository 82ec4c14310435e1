set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
PDG_A_SOLVER=local PDG_FLOW_SOLVER=blocktri timeout 600 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench_blocktri.json 2> gpurun_out/bench_blocktri.err; echo "bench bt rc $?"
timeout 300 python tools/debug_nd.py 128 > gpurun_out/nd_debug.log 2>&1; echo "dbg rc $?"
