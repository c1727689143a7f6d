mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/peaks scripts/ubench/peaks.cu && /tmp/peaks > gpurun_out/r02b_peaks.json; cat gpurun_out/r02b_peaks.json
bash scripts/gpu_variants.sh 2>&1 | tee gpurun_out/r02b_variants.txt
timeout 1200 python -m pytest tests/test_gpu_instances.py tests/test_gpu_taps.py tests/test_gpu_reference_suite.py tests/test_gpu_shard.py tests/test_gpu_plugin.py -q -x -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02b_pytest.log
