set -x
CF_NO_ST16T=1 timeout 300 python scripts/st16t_ab.py 2>&1 | tail -2
for S in 4 3 6; do CF_ST16T_STAGES=$S timeout 300 python scripts/st16t_ab.py 2>&1 | tail -2; done
timeout 900 python -m pytest tests -m gpu -x -q -k "48 or 64 or lane or stencil or vcycle or slab" 2>&1 | tail -5
