#!/bin/bash
# full ncu captures of the grouped SpGEMM numeric kernel of one config-3 u-hierarchy build
mkdir -p gpurun_out
python scripts/ncu_amg.py > gpurun_out/ncu_amg_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_num_grp -c 2 \
    -o gpurun_out/prof_numgrp3 python scripts/ncu_amg.py > gpurun_out/ncu_grp.log 2>&1
echo grp rc=$?
