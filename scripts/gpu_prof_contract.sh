# ncu --set full of the two K2 forms on the bench workload (40 frames): the
# FP32-FMA symmetric kernel and the tcgen05 3xTF32 kernel (KKB_CONTRACT=tc)
CMD="python bench.py --frames 40 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/pc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_contract" -s 3 -c 1 -f -o gpurun_out/prof_contract_fma $CMD > gpurun_out/ncu_c1.log 2>&1
echo "fma rc=$?"
KKB_CONTRACT=tc $CMD > gpurun_out/pc_plain2.log 2>&1 && \
KKB_CONTRACT=tc ncu --set full --clock-control none --import-source on -k regex:"k_contract" -s 3 -c 1 -f -o gpurun_out/prof_contract_tc $CMD > gpurun_out/ncu_c2.log 2>&1
echo "tc rc=$?"
