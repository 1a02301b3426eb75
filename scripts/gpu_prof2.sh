# config-3 step: per-kernel device time, per-phase AMG build split, hierarchy build timings
mkdir -p gpurun_out
bash scripts/gpu_profile.sh
CF_TIMING=1 timeout 600 python scripts/amg_build_profile.py > gpurun_out/amg_build_profile.txt 2> gpurun_out/amg_build_timing.log; echo abp rc=$?
