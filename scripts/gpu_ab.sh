timeout 600 python scripts/residual_ab.py 2>&1 | grep residual
CF_LIB_PATH=build_ab/lib_plaindiv.so timeout 600 python scripts/residual_ab.py 2>&1 | grep residual
