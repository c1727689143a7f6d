# launch list + full ncu capture of the hot kernels (small config-4 batch)
CMD="python bench.py --frames 40 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kk_gather|k_contract|k_fft_r2c|k_fft_c2c" -s 12 -c 4 -o gpurun_out/prof_r1a $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -5 gpurun_out/ncu_full.log
