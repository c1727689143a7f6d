# scaling prediction + launch list + ncu --set full of the five step kernels
mkdir -p gpurun_out
timeout 600 python scripts/scaling_predict.py gpurun_out/r02_scaling.json > gpurun_out/r02f_scaling.log 2>&1; echo "scaling rc=$?"; tail -3 gpurun_out/r02f_scaling.log
bash scripts/gpu_prof_round.sh launches; echo "launches rc=$?"
bash scripts/gpu_prof_final.sh step; echo "full rc=$?"
ls -la gpurun_out/*.ncu-rep 2>/dev/null
