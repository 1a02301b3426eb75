set -x
timeout 300 python scripts/mf_ab.py 2>&1 | grep cfg
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_parity_large.py tests/test_gpu_multirank.py tests/test_gpu_slab.py -m gpu -x -q -k "matrix_free or mf or multirank or slab or nccl" 2>&1 | tail -3
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
