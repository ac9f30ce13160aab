timeout 2400 python tools/calibrate.py measure --only-new --out gpurun_out/calib_raw_r2c.json > gpurun_out/calib_measure3.log 2>&1
tail -1 gpurun_out/calib_measure3.log
