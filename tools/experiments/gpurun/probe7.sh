timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2b.log 2>&1
tail -3 gpurun_out/gpu_tests_r2b.log
timeout 2400 python tools/calibrate.py measure --out gpurun_out/calib_raw_r2.json > gpurun_out/calib_measure.log 2>&1
tail -2 gpurun_out/calib_measure.log
