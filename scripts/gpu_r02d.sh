mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_media.py -q -x -p no:cacheprovider > gpurun_out/r02d_media.log 2>&1; echo "media rc=$?"; tail -15 gpurun_out/r02d_media.log
timeout 600 python scripts/dropin_latency.py gpurun_out/r02d_dropin.json > gpurun_out/r02d_dropin.log 2>&1; echo "dropin rc=$?"; cat gpurun_out/r02d_dropin.log | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/r02d_bench.json
