timeout 900 python scripts/level_spmv.py > gpurun_out/level_spmv.txt 2>&1; echo lv rc=$?
CF_VCYCLE_UNFUSED=1 timeout 900 python scripts/level_spmv.py --quick > gpurun_out/level_spmv_unfused.txt 2>&1; echo lvu rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "amg or vcycle or solver" > gpurun_out/gpu_tests_amg.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_amg.log
