L=build_ab/lib_lowhash.so
timeout 600 python scripts/amg_build_ab.py 2>&1 | grep hierarchy | sed 's/^/high /'
CF_LIB_PATH=$L timeout 600 python scripts/amg_build_ab.py 2>&1 | grep hierarchy | sed 's/^/low /'
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
