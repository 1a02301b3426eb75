for pf in 0 2 3 7; do
  echo "CF_SPMV_PF=$pf"; CF_SPMV_PF=$pf timeout 300 python scripts/vcycle_profile.py 2>&1 | grep -E "V-cycle kernel total|k_spmv_b|k_spmv_pf" | head -8
  CF_SPMV_PF=$pf timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],1), d['phase_ms_last_step'], d['vcycle']['u_ms'], d['vcycle']['phi_ms'])"
done
