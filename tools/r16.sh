timeout 300 python tools/nd_once2.py > gpurun_out/nd_once2.log 2>&1; echo "once rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve --launch-skip 3 -c 1 -o gpurun_out/nd_full3 -f python tools/nd_once2.py > gpurun_out/ncu_nd3.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/nd_full3.ncu-rep --page source --csv --print-source sass > gpurun_out/nd_src_sass.csv 2>&1
ncu -i gpurun_out/nd_full3.ncu-rep --page source --csv --print-source cuda > gpurun_out/nd_src_cuda.csv 2>&1
ncu -i gpurun_out/nd_full3.ncu-rep --page details > gpurun_out/nd_details.txt 2>&1
ls -la gpurun_out
