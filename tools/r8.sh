set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve --launch-skip 8 -c 4 -o gpurun_out/nd_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --spmv-sizes "" > gpurun_out/ncu_nd.log 2>&1; echo "ncu rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --spmv-sizes "" > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
