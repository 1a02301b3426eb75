for v in "" "CF_SPGEMM_NO_RUNS=1"; do
  echo "== $v"
  env $v timeout 300 python scripts/amg_build_profile.py u 2>&1 | grep -E "u-build|k_num_grp" | head -6
  env $v timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],1), d['phase_ms_last_step'])"
done
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_parity_large.py -x -q -k "amg or hierarchy or 48 or 64 or grouped or paths" 2>&1 | tail -2
