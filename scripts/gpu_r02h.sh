# round-2 re-entry validation: smoke, GPU suite, bench, AMG phase breakdown, kernel profile
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
CF_TIMING=1 timeout 600 python scripts/step_phases.py 2> gpurun_out/phases.log; python scripts/step_phases.py --parse gpurun_out/phases.log > gpurun_out/phases.txt; tail -80 gpurun_out/phases.txt
timeout 600 python scripts/kernel_profile.py > gpurun_out/kernel_profile.txt 2>&1; head -50 gpurun_out/kernel_profile.txt
