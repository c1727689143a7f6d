# ncu of the tensor-core gather (config 4, 400 frames): launch list of the
# check script, then --set full of the first k_kk_gather_tc launch
python scripts/tc_gather_check.py > gpurun_out/tcg_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/tcg_launches.csv \
    python scripts/tc_gather_check.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kk_gather_tc" -c 1 -f -o gpurun_out/prof_tcg python scripts/tc_gather_check.py > gpurun_out/ncu_tcg.log 2>&1
echo "rc=$?"
