for g in 16 32 48 8; do
  echo "=== group $g"
  VX_GROUP_P=$g python tools/cublas_vs_ours.py 16383,12288,4096 16384,11008,4096 8192,4096,4096 4096,11008,4096 2>&1 | grep -v cublas_probe
done > gpurun_out/group_probe.txt 2>&1
for g in 16 32; do
  VX_GROUP_P=$g ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:vx_umma -s 2 -c 1 python tools/launch_n.py 16383 12288 4096 --R 4 2>&1 | grep -E "dram__|gpu__time" >> gpurun_out/group_probe.txt
done
VX_GROUP_P=32 timeout 900 python -m pytest tests -x -q -m gpu -k "every_rung or full_schedule or deep_k" > gpurun_out/group_tests.log 2>&1; tail -1 gpurun_out/group_tests.log
