T="python tools/timeline.py 128 3072 768"
( echo "=== base"; $T
  echo "=== dbg8 (no epilogue stores)"; VX_DEBUG_FLAGS=8 $T
  echo "=== dbg128 (no L2 prefetch)"; VX_DEBUG_FLAGS=128 $T
  echo "=== dbg512 (no MMA)"; VX_DEBUG_FLAGS=512 $T
  echo "=== nopdl"; VX_PDL=0 $T
  echo "=== swap128x32 s1"; python tools/timeline.py 128 3072 768 6 1
  echo "=== swap128x16 s1"; python tools/timeline.py 128 3072 768 5 1
  echo "=== swap128x64 s1"; python tools/timeline.py 128 3072 768 7 1
) > gpurun_out/probe5.txt 2>&1
