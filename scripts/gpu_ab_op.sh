#!/bin/bash
# A/B: phi rows of the Krylov operator on the auxiliary stream (default) vs one stream
mkdir -p gpurun_out
for v in "CF_SERIAL_OPERATOR=1" ""; do
  echo "== $v"
  env $v timeout 600 python bench.py --no-cpu --no-operator --no-rebuild-check --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],1), d['phase_ms_last_step'], d['ms_each_step'])"
done
CF_TIMING=1 python scripts/step_phases.py 2> gpurun_out/phases_r02h.log > /dev/null
awk '/@@STEP2@@/{f=1} f' gpurun_out/phases_r02h.log | grep "L0\] \(n2\|S^T\)"
