set -x
mkdir -p gpurun_out
python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r01_cfg3.csv python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton.log 2>&1
echo launches rc=$?
python scripts/ncu_operator.py > gpurun_out/ncu_op_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmv_b -s 1 -c 1 \
    -o gpurun_out/prof_r01_spmv_cfg1 python scripts/ncu_operator.py > gpurun_out/ncu_op.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_newton.log gpurun_out/ncu_op.log
