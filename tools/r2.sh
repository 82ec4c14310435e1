set -x
timeout 300 python tools/debug_nd.py 128 > gpurun_out/nd_debug.log 2>&1; echo "dbg rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve -c 4 -o gpurun_out/nd_full python tools/nd_once.py 128 > gpurun_out/ncu_nd.log 2>&1; echo "ncu rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --spmv-sizes 256 --spmv-reps 3 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
