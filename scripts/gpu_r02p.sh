set -x
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_reuse.py tests/test_gpu_parity_large.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
CF_SPGEMM_SMALL_ROWS=32768 timeout 300 python scripts/step_series.py 3 2>&1 | head -5
CF_SPGEMM_NO_STAGED=1 timeout 300 python scripts/step_series.py 3 2>&1 | head -5
