timeout 300 python tools/nd_once2.py > gpurun_out/nd_once2.log 2>&1; echo "once rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nd_solve --launch-skip 2 -c 2 -o gpurun_out/nd_full2 -f python tools/nd_once2.py > gpurun_out/ncu_nd2.log 2>&1; echo "ncu rc $?"
