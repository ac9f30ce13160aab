ncu --set full --clock-control none --import-source on -k regex:vx_umma -s 6 -c 1 -o gpurun_out/bert128 -f python tools/launch_n.py 128 3072 768 > gpurun_out/probe3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vx_umma -s 6 -c 1 -o gpurun_out/split4 -f python tools/launch_n.py 128 1024 1024 0 4 >> gpurun_out/probe3.log 2>&1
