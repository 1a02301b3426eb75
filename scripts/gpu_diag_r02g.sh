#!/bin/bash
# round-2 (session 3) diagnosis: AMG build phases, kernel breakdown of a warm config-3 step,
# phi-build breakdown at the converged state, and a bounded compute-sanitizer attempt.
mkdir -p gpurun_out
CF_TIMING=1 python scripts/step_phases.py 2> gpurun_out/phases_r02g.log > /dev/null
python scripts/step_phases.py --parse gpurun_out/phases_r02g.log > gpurun_out/phases_r02g.txt
TOPN=60 python scripts/kernel_profile.py cfg3 20 > gpurun_out/kernel_profile_r02g.txt 2>&1
python scripts/phi_build_profile.py > gpurun_out/phi_build_r02g.txt 2>&1
SAN_TIMEOUT=300 bash scripts/gpu_sanitize.sh 4 2
