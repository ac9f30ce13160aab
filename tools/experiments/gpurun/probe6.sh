timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_mc.log 2>&1
tail -5 gpurun_out/gpu_tests_mc.log
( for f in "1 1" "2 1" "10 1" "11 1" "12 1" "9 1"; do echo "=== rung $f"; timeout 120 python tools/timeline.py 128 3072 768 $f; done
  echo "=== 512x768 rung 2"; timeout 120 python tools/timeline.py 512 768 768 2 1
  echo "=== 512x768 rung 1"; timeout 120 python tools/timeline.py 512 768 768 1 1
) > gpurun_out/probe6.txt 2>&1
