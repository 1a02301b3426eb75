timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python scripts/kernel_profile.py cfg3 20 > gpurun_out/kernel_profile.txt 2>&1; echo kp rc=$?
