timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_lean.log 2>&1
tail -3 gpurun_out/gpu_tests_lean.log
( for sh in "128 3072 768" "384 3072 768" "512 2304 768" "1024 768 768" "64 2304 768"; do
    for f in "0 1" "1 1" "11 1" "12 1" "14 1" "15 1"; do
      echo "=== $sh rung $f"; timeout 120 python tools/timeline.py $sh $f 2>&1 | grep -E "per-launch|acc_ready|exit "
    done
  done ) > gpurun_out/probe19.txt 2>&1
