CF_SPGEMM_GRP_V1=1 timeout 600 python scripts/amg_build_ab.py > gpurun_out/plain_v1.log 2>&1 && \
CF_SPGEMM_GRP_V1=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_num_grp -c 4 -o gpurun_out/grp_v1 python scripts/amg_build_ab.py > gpurun_out/ncu_v1.log 2>&1; echo v1 rc=$?
timeout 600 python scripts/amg_build_ab.py > gpurun_out/plain_pf.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_num_grp -c 4 -o gpurun_out/grp_pf python scripts/amg_build_ab.py > gpurun_out/ncu_pf.log 2>&1; echo pf rc=$?
