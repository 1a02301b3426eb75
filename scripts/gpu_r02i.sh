set -x
CF_NO_ST16T=1 timeout 300 python scripts/st16t_ab.py 2>&1 | tail -1
for S in 3 2 4; do CF_ST16T_STAGES=$S timeout 300 python scripts/st16t_ab.py 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gpu_tests.log
CF_AMG_NO_COMPACT=1 timeout 300 python scripts/step_series.py 3 2>&1 | head -5
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
