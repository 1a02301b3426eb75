set -x
timeout 300 python scripts/step_series.py 3 2>&1 | head -5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
python scripts/ncu_operator.py > gpurun_out/op_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmv_st16t -s 1 -c 1 \
    -o gpurun_out/prof_r02_st16t python scripts/ncu_operator.py > gpurun_out/ncu_op.log 2>&1
echo st16t rc=$?
ncu -i gpurun_out/prof_r02_st16t.ncu-rep --page raw --csv > gpurun_out/prof_r02_st16t_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02_st16t.ncu-rep --page details --csv > gpurun_out/prof_r02_st16t_details.csv 2>/dev/null
ls -la gpurun_out/
