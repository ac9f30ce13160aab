set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/timeline.py 128 3072 768 > gpurun_out/tl_128_3072_768.txt 2>&1
python tools/timeline.py 16 1536 512 5 4 > gpurun_out/tl_16_1536_512_s4.txt 2>&1
python tools/timeline.py 128 1024 1024 0 4 > gpurun_out/tl_128_1024_1024_u64s4.txt 2>&1
python tools/timeline.py 128 1024 1024 0 1 > gpurun_out/tl_128_1024_1024_u64s1.txt 2>&1
python tools/timeline.py 512 768 768 > gpurun_out/tl_512_768_768.txt 2>&1
python tools/timeline.py 16 11008 4096 > gpurun_out/tl_16_11008_4096.txt 2>&1
python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2_start.log 2>&1
tail -3 gpurun_out/gpu_tests_r2_start.log
