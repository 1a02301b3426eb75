timeout 300 python scripts/spmv_ab.py 2>&1 | grep -v Warn
CF_CSR_NOPF=1 timeout 300 python scripts/spmv_ab.py 2>&1 | grep -v Warn | grep csr
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python scripts/kernel_profile.py cfg3 50 > gpurun_out/kprof.log 2>&1; head -3 gpurun_out/kprof.log | tail -2
