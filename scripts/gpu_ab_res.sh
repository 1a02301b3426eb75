for L in build_ab/lib_resminb3.so build_ab/lib_head.so build_ab/lib_resminb4.so; do
CF_LIB_PATH=$L timeout 300 python scripts/residual_ab.py 2>&1 | grep residual
done
