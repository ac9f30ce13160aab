timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2g.log 2>&1
tail -2 gpurun_out/gpu_tests_r2g.log
python bench.py --steps 10 --warmup 3 --points-out gpurun_out/bench_points_r2d.json > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
tail -c 300 gpurun_out/bench_r2d.err
mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:vx_umma -s 2 -c 1 -o gpurun_out/ncu/r02_dominant -f python tools/launch_n.py 16383 12288 4096 --R 4 > gpurun_out/ncu/dom.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vx_umma -s 4 -c 1 -o gpurun_out/ncu/r02_bert -f python tools/launch_n.py 128 3072 768 --R 8 > gpurun_out/ncu/bert.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vx_ -s 4 -c 1 -o gpurun_out/ncu/r02_decode16 -f python tools/launch_n.py 16 11008 4096 --R 8 > gpurun_out/ncu/dec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vx_umma -s 4 -c 1 -o gpurun_out/ncu/r02_mc2 -f python tools/launch_n.py 128 11008 4096 --R 8 > gpurun_out/ncu/mc2.log 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/ncu/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-cublas --no-extra > gpurun_out/ncu/launches_bench.log 2>&1
ls -la gpurun_out/ncu
