timeout 3000 python tools/sweep.py --shapes all --method graph --reps 3 --out gpurun_out/heldout_sweep_r2.json > gpurun_out/heldout_sweep.log 2>&1
tail -3 gpurun_out/heldout_sweep.log
