for v in "" "CF_NO_PREC_GRAPH=1"; do
  echo "== $v"
  env $v timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],1), d['ms_each_step'], d['phase_ms_last_step'], d['gpu_launches_per_step'])"
done
timeout 1200 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_solver.py tests/test_gpu_reuse.py -x -q 2>&1 | tail -2
