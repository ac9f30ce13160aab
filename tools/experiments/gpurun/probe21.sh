timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2f.log 2>&1
tail -3 gpurun_out/gpu_tests_r2f.log
