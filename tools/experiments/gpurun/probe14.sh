timeout 1500 python -m pytest tests -x -q -m gpu -rs > gpurun_out/gpu_tests_r2d.log 2>&1
tail -5 gpurun_out/gpu_tests_r2d.log
timeout 900 python tools/analyzer_ablation.py measure --out-dir gpurun_out > gpurun_out/ablation_measure.log 2>&1
cat gpurun_out/ablation_measure.log
