timeout 900 python bench.py --points-out gpurun_out/points48.json --no-e2e > gpurun_out/bench48.log 2>&1; echo bench=$?
