timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2e.log 2>&1
tail -3 gpurun_out/gpu_tests_r2e.log
python tools/m16probe.py > gpurun_out/m16b.txt 2>&1
VX_DEBUG_FLAGS=65536 python tools/m16probe.py >> gpurun_out/m16b.txt 2>&1
