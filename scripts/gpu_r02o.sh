# full validation of the round-2 re-entry state: smoke, GPU suite, bench (+ reference arm), ncu launch list
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02h_cfg3.csv python scripts/ncu_newton.py 2 > gpurun_out/ncu_newton.log 2>&1
echo launches rc=$?
