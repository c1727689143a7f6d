# full ncu capture of the stage-1 kernels (real FFT, contraction, inverse FFT)
CMD="python bench.py --frames 40 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plainF.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_r2c|k_contract|k_c2c" -s 6 -c 3 -f -o gpurun_out/prof_fft $CMD > gpurun_out/ncu_fft.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_fft.log
