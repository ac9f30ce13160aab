python bench.py --steps 10 --warmup 3 --points-out gpurun_out/bench_points_r2c.json > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
tail -c 400 gpurun_out/bench_r2c.err
timeout 3000 python tools/sweep.py --shapes all --method graph --reps 3 --out gpurun_out/heldout_sweep_r2c.json > gpurun_out/heldout_sweep_c.log 2>&1
tail -1 gpurun_out/heldout_sweep_c.log
