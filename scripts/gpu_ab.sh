for L in default build_ab/lib_head.so default build_ab/lib_head.so; do
if [ $L = default ]; then unset CF_LIB_PATH; else export CF_LIB_PATH=$L; fi
timeout 600 python scripts/amg_build_ab.py 2>&1 | grep hierarchy | sed "s|^|$L |"
done
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k "amg or block_prec or penny" > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t.log
