CF_NO_STENCIL_COLS=1 timeout 300 python scripts/spmv_ab.py 2>&1 | grep -v Warn | grep csr
CF_CSR_V1=1 CF_NO_STENCIL_COLS=1 timeout 300 python scripts/spmv_ab.py 2>&1 | grep -v Warn | grep csr
timeout 600 python scripts/kernel_profile.py cfg3 50 2>&1 | grep -E "^\{|total|spmv_b"
CF_CSR_V1=1 timeout 600 python scripts/kernel_profile.py cfg3 50 2>&1 | grep -E "^\{|total|spmv_b"
