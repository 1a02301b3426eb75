# round-2 diagnostics: AMG build phases with N2 tier counts; ncu captures of the residual kernel and
# the level-0 SpGEMM numeric (k_num_grp<4>) inside a config-3 step.
mkdir -p gpurun_out
make -s -j8 -C paper_1806_09924_b200/csrc >/dev/null
CF_TIMING=1 timeout 600 python scripts/step_phases.py 2> gpurun_out/step_phases.log > /dev/null; echo sp rc=$?
python scripts/ncu_newton.py 1 > gpurun_out/nn_plain.log 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" -k regex:k_cell_residual_q -c 1 \
    -o gpurun_out/prof_r02b_residual python scripts/ncu_newton.py 1 > gpurun_out/ncu_res.log 2>&1; echo res rc=$?
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" -k regex:k_num_grp -c 1 \
    -o gpurun_out/prof_r02b_numgrp python scripts/ncu_newton.py 1 > gpurun_out/ncu_grp.log 2>&1; echo grp rc=$?
