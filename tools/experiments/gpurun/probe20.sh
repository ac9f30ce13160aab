timeout 3000 python tools/calibrate.py measure --out gpurun_out/calib_raw_r2d.json > gpurun_out/calib_measure4.log 2>&1
tail -1 gpurun_out/calib_measure4.log
