for L in default build_ab/lib_plaindiv.so; do
if [ $L = default ]; then unset CF_LIB_PATH; else export CF_LIB_PATH=$L; fi
timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 2 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],1), d['phase_ms_last_step'])"
done
