for v in "" "CF_SPMV_NOGROUP=1" "CF_QPSTATE_SERIAL=1"; do
  echo "== $v"; env $v timeout 300 python scripts/vcycle_profile.py 2>&1 | grep -E "V-cycle kernel total|k_spmv_grp|k_spmv_b<8" | head -4
  env $v timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],1), d['phase_ms_last_step'], d['vcycle']['u_ms'])"
done
timeout 1200 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_solver.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
