python bench.py --steps 10 --warmup 3 --points-out gpurun_out/bench_points_r2a.json > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -c 3000 gpurun_out/bench_r2a.json
