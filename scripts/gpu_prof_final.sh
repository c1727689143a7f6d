# Final-round ncu captures (one ncu per call is the rule; pass the target):
#   step  -> the five kernels of one bench step (config 4, 400 frames)
#   das   -> the tiled DAS kernel on the config-2 DAS workload
case "$1" in
  step)
    CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
    $CMD > gpurun_out/prof_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_kk_gather|k_r2c|k_contract|k_c2c|k_log_compress" -s 15 -c 5 -f -o gpurun_out/prof_final_step $CMD > gpurun_out/ncu_final.log 2>&1 ;;
  das)
    CMD="python scripts/das_bench.py"
    $CMD > gpurun_out/prof_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k_das_tile -c 1 -f -o gpurun_out/prof_final_das $CMD > gpurun_out/ncu_final.log 2>&1 ;;
esac
echo "ncu rc=$?"
