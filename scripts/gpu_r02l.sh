set -x
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_reuse.py tests/test_gpu_parity_large.py -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
CF_TIMING=1 timeout 600 python scripts/step_phases.py 2> gpurun_out/phases3.log; python scripts/step_phases.py --parse gpurun_out/phases3.log > gpurun_out/phases3.txt; tail -3 gpurun_out/phases3.txt
timeout 600 python scripts/level_spmv.py --quick > gpurun_out/level_spmv.txt 2>&1; tail -40 gpurun_out/level_spmv.txt
