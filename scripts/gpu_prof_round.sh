# Round profile of the bench default (config 4, 400 frames): $1 = "launches" or "full"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/prof_plain.log; exit 1; }
if [ "$1" = launches ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
else
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_kk_gather|k_r2c|k_contract|k_c2c|k_log_compress|k_split_planes|k_frame_maxabs" -s 24 -c 8 -f -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
fi
echo "ncu rc=$?"
