#!/bin/bash
# A/B of the SpGEMM L2 hints (CF_SPGEMM_HINT 0/1/2): config-3 u-hierarchy build time and level hash
mkdir -p gpurun_out
for v in h0 h1 default; do
  if [ $v = default ]; then L=""; else L="CF_LIB_PATH=build_ab/lib_$v.so"; fi
  echo "== $v"
  env $L timeout 300 python scripts/amg_ab.py cfg3 2>&1 | head -14
done
