# kernel/phase breakdowns of the config-3 step (torch profiler; CF_TIMING phases)
timeout 600 python scripts/vcycle_profile.py > gpurun_out/vcycle_profile.txt 2>&1; echo vc rc=$?
timeout 600 python scripts/kernel_profile.py cfg3 20 > gpurun_out/kernel_profile.txt 2>&1; echo kp rc=$?
CF_TIMING=1 timeout 600 python scripts/step_phases.py 2> gpurun_out/step_phases.log > /dev/null; echo sp rc=$?
python scripts/step_phases.py --parse gpurun_out/step_phases.log > gpurun_out/step_phases.txt 2>&1
