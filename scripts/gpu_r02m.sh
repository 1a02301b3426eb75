set -x
CF_NO_SPMV_BT=1 timeout 600 python scripts/level_spmv.py --quick 2>&1 | grep "u L0 P\|u L1 P\|V-cycle"
timeout 600 python scripts/level_spmv.py --quick 2>&1 | grep "u L0 P\|u L1 P\|V-cycle"
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_reuse.py tests/test_gpu_parity_large.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
