timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err; echo "ref rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --spmv-sizes '' > gpurun_out/g_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve --launch-skip 2 -c 2 -o gpurun_out/g_nd_full -f python tools/nd_once2.py > gpurun_out/g_ncu_nd.log 2>&1; echo "ncu nd rc $?"
ncu -i gpurun_out/g_nd_full.ncu-rep --page details > gpurun_out/g_nd_details.txt 2>&1
ncu -i gpurun_out/g_nd_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/g_nd_dram.csv 2>&1
