set -x
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_reuse.py tests/test_gpu_parity_large.py -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
timeout 600 python scripts/gpu_timeline.py > gpurun_out/timeline2.txt 2>&1; sed -n 3,34p gpurun_out/timeline2.txt
