timeout 600 python scripts/amg_build_ab.py 2>&1 | grep hierarchy
CF_LIB_PATH=build_ab/lib_head.so timeout 600 python scripts/amg_build_ab.py 2>&1 | grep hierarchy
