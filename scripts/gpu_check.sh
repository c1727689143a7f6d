# tests + smoke + bench + launch list (exact bench command) + ncu of the hot kernels
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "${PROFILE:-1}" = "1" ]; then
python bench.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kk_gather" -s 3 -c 1 -f -o gpurun_out/prof_gather $CMD > gpurun_out/ncu_full.log 2>&1
echo "full gather rc=$?"
CMD="python bench.py --frames 40 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_contract|k_r2c|k_c2c|k_log" -s 12 -c 4 -f -o gpurun_out/prof_stage1 $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full stage1 rc=$?"
fi
