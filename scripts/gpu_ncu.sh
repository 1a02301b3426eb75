# ncu evidence for profiles/: launch list of the first two Newton iterations of a config-3 step and
# full captures of the stencil SpMV (config 1 M_uu, the roofline kernel) and of the largest SpGEMM
# numeric launch of the u-hierarchy build.  usage: bash scripts/gpu_ncu.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_cfg3.csv python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton.log 2>&1
echo launches rc=$?
python scripts/ncu_operator.py > gpurun_out/op_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmv_st16p -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_st16p python scripts/ncu_operator.py > gpurun_out/ncu_op.log 2>&1
echo st16p rc=$?
python scripts/amg_build_ab.py > gpurun_out/amg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_num_grp -c 1 \
    -o gpurun_out/prof_${TAG}_numgrp python scripts/amg_build_ab.py > gpurun_out/ncu_amg.log 2>&1
echo numgrp rc=$?
