timeout 600 python scripts/assembly_bench.py cfg3 > gpurun_out/asm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_jac_fill_pair|k_cell_residual_q" -c 2 -o gpurun_out/asm python scripts/assembly_bench.py cfg3 > gpurun_out/ncu_asm.log 2>&1; echo rc=$?
cat gpurun_out/asm_plain.log | grep -v Warn
