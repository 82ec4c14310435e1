timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config0_parity or restart" > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc $?"
for L in 64 128 192 256 384; do echo "=== flow leaf $L"; PDG_ND_FLOW_LEAF=$L timeout 120 python tools/debug_nd.py 128 2>&1 | grep "nd solve n=33024" | sed 's/fronts.*total/total/'; done > gpurun_out/flow_leaf.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo "bench rc $?"
PDG_KRYLOV_UNFUSED=1 timeout 900 python bench.py --no-cpu-baseline --spmv-sizes 256 > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err; echo "bench rc $?"
