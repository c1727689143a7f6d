mkdir -p gpurun_out
for v in default c2c3 default c2c3; do
  if [ $v = default ]; then unset KKB_LIB; else export KKB_LIB=$PWD/paper_2603_22496_b200/variants/libkkb_$v.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_sequential'])" >> gpurun_out/exp_k3.txt
done
export KKB_LIB=$PWD/paper_2603_22496_b200/variants/libkkb_c2c3.so
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_fused_tc.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/exp_k3.txt
unset KKB_LIB
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches_bench_default.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02h_ncu.log 2>&1
cat gpurun_out/exp_k3.txt
