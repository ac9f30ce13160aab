for f in 0 1024 2048; do
  echo "=== flags $f cold"; VX_DEBUG_FLAGS=$f python tools/timeline.py 128 3072 768
  echo "=== flags $f hot"; VX_DEBUG_FLAGS=$f python tools/timeline.py 128 3072 768 --hot
done > gpurun_out/probe2.txt 2>&1
for f in 0 1024; do
  echo "=== split4 flags $f cold"; VX_DEBUG_FLAGS=$f python tools/timeline.py 128 1024 1024 0 4
  echo "=== split4 flags $f hot"; VX_DEBUG_FLAGS=$f python tools/timeline.py 128 1024 1024 0 4 --hot
done > gpurun_out/probe2b.txt 2>&1
