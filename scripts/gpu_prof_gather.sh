CMD="python bench.py --frames 40 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plainG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kk_gather" -s 3 -c 1 -f -o gpurun_out/prof_g2 $CMD > gpurun_out/ncu_g2.log 2>&1
echo "rc=$?"
