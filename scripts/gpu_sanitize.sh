#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on one 48^3 penny Newton step
# (the 16-lane stencil SpMVs, the Jacobian fill, the AMG setup and V-cycles, GMRES).
# OPKIND=1 (default) runs the matrix-free operator, 0 the assembled one.
# Logs: gpurun_out/sanitizer_<tool>.log; summaries are copied to profiles/ by hand.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
N=${1:-12}; R=${2:-2}
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout ${SAN_TIMEOUT:-1200} $CS --tool $tool $extra --print-limit 50 --error-exitcode 99 \
    env CF_RUNNER_OPKIND=${OPKIND:-1} python tests/_newton_runner.py 3 $N $R 1 > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_$tool.log >> gpurun_out/sanitizer_summary.txt
done
