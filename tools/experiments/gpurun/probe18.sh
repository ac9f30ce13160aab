timeout 1500 python -m pytest tests -x -q -m gpu -k "full_schedule" > gpurun_out/gpu_tests_fullsched.log 2>&1
tail -3 gpurun_out/gpu_tests_fullsched.log
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; tail -3 gpurun_out/sanitize_plain.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -4 gpurun_out/sanitize_$t.log
done
