set -x
timeout 600 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k "empty_coarse or amg" 2>&1 | tail -5
CF_TIMING=1 timeout 600 python scripts/step_phases.py 2> gpurun_out/phases2.log; python scripts/step_phases.py --parse gpurun_out/phases2.log > gpurun_out/phases2.txt; tail -3 gpurun_out/phases2.txt
