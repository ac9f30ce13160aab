python tools/m16probe.py > gpurun_out/m16.txt 2>&1
VX_DEBUG_FLAGS=4096 python tools/m16probe.py >> gpurun_out/m16.txt 2>&1
VX_DEBUG_FLAGS=128 python tools/m16probe.py >> gpurun_out/m16.txt 2>&1
VX_DEBUG_FLAGS=2048 python tools/m16probe.py >> gpurun_out/m16.txt 2>&1
