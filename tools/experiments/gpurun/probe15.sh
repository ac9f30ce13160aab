python bench.py --steps 10 --warmup 3 --points-out gpurun_out/bench_points_r2b.json > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
timeout 3000 python tools/sweep.py --shapes all --method graph --reps 3 --out gpurun_out/heldout_sweep_r2b.json > gpurun_out/heldout_sweep_b.log 2>&1
