# A/B of the matrix-free sweep's tile size (owned vertices per side _ min CTAs per SM)
for v in 8_5 7_8 10_4 10_3; do CF_LIB_PATH=build_ab/lib_mf$v.so timeout 300 python scripts/mf_ab.py 2>&1 | grep "cfg"; done
