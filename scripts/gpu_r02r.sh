set -x
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
