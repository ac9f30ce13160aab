timeout 900 python -m pytest tests -x -q -m gpu -k "every_rung or pdl or pad_poison or deep_k" > gpurun_out/gpu_tests_pair64.log 2>&1
tail -3 gpurun_out/gpu_tests_pair64.log
( for s in "128 3072 768" "512 768 768" "512 3072 768" "1024 3072 768" "256 2304 768" "1024 768 768"; do
    echo "=== $s pair64"; timeout 120 python tools/timeline.py $s 6 1 | grep -E "per-launch|acc_ready|epi_done|first_full|exit "
    echo "=== $s selected"; timeout 120 python tools/timeline.py $s | grep -E "per-launch|exit "
  done ) > gpurun_out/probe9.txt 2>&1
timeout 2400 python tools/calibrate.py measure --out gpurun_out/calib_raw_r2b.json > gpurun_out/calib_measure2.log 2>&1
tail -1 gpurun_out/calib_measure2.log
