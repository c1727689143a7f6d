# Round-2 final evidence for the bench default (config 4, 400 frames):
#   bench   -> one bench.py line (gpurun_out/${R:-r02e}_bench.log)
#   launch  -> ncu launch list of a short bench run (per-launch durations)
#   full    -> ncu --set full of the six kernels of one step (after warm-up)
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
case "$1" in
  bench)
    python bench.py > gpurun_out/${R:-r02e}_bench.log 2>&1 ;;
  launch)
    $CMD > gpurun_out/prof_plain.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R:-r02e}_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ;;
  full)
    $CMD > gpurun_out/prof_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_kk_gather_tc|k_r2c|k_contract_sym|k_c2c_planes|k_frame_bound|k_log_compress" -s 18 -c 6 -f \
        -o gpurun_out/${R:-r02e}_step $CMD > gpurun_out/ncu_full.log 2>&1 ;;
esac
echo "$1 rc=$?"
