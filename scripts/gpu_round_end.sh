timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 2400 bash scripts/gpu_ncu.sh ${1:-r01d}
