timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve --launch-skip 3 -c 1 -o gpurun_out/nd_full4 -f python tools/nd_once2.py > gpurun_out/ncu_nd4.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/nd_full4.ncu-rep --page source --csv --print-source sass > gpurun_out/nd4_sass.csv 2>&1
ncu -i gpurun_out/nd_full4.ncu-rep --page details > gpurun_out/nd4_details.txt 2>&1
ncu -i gpurun_out/nd_full4.ncu-rep --page raw --csv > gpurun_out/nd4_raw.csv 2>&1
