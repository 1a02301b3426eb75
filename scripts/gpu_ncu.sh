# ncu evidence for profiles/: launch list of two config-3 Newton iterations, full captures of the
# stencil SpMV (config 1) and the Jacobian fill.  usage: bash scripts/gpu_ncu.sh TAG
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_cfg3.csv python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton.log 2>&1
echo launches rc=$?
python scripts/ncu_asm.py > gpurun_out/asm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_jac_fill_pair -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_jacfill python scripts/ncu_asm.py > gpurun_out/ncu_asm.log 2>&1
echo jac rc=$?
tail -2 gpurun_out/ncu_newton.log gpurun_out/ncu_asm.log
