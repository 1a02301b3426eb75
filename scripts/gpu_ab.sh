for L in build_ab/lib_new.so build_ab/lib_head.so; do
CF_LIB_PATH=$L timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],1), d['phase_ms_last_step'])"
done
for L in build_ab/lib_new.so build_ab/lib_head.so; do
CF_LIB_PATH=$L timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],1), d['phase_ms_last_step'])"
done
CF_LIB_PATH=build_ab/lib_new.so timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_multirank.py -x -q -k "not forced and not everywhere" > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t.log
