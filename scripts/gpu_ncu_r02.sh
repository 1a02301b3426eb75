# round-2 ncu evidence: launch list of the first two Newton iterations of a config-3 step, full
# captures of the matrix-free sweep (config 3, inside the step) and of the config-1 stencil SpMV
mkdir -p gpurun_out
python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02_cfg3.csv python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" -k regex:k_mf_sweep -c 1 \
    -o gpurun_out/prof_r02_mf_sweep python scripts/ncu_newton.py 1 > gpurun_out/ncu_mf.log 2>&1
echo mf rc=$?
python scripts/ncu_operator.py > gpurun_out/op_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmv_st16p -s 1 -c 1 \
    -o gpurun_out/prof_r02_st16p python scripts/ncu_operator.py > gpurun_out/ncu_op.log 2>&1
echo st16p rc=$?
