# ncu --set full of the tensor-core gather (config 4, 64 frames)
python scripts/tc_gather_check.py > gpurun_out/tcg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kk_gather_tc" -c 1 -f -o gpurun_out/prof_tcg python scripts/tc_gather_check.py > gpurun_out/ncu_tcg.log 2>&1
echo "rc=$?"
