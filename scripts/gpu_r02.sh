# Round-2 GPU check: smoke, the -m gpu suite, bench, on-chip peak ubench,
# K5 instance sweep.  Usage: bash scripts/gpu_r02.sh [TAG]
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest_gpu.log
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | head -c 3000; tail -3 gpurun_out/${TAG}_bench.err
fi
if [ "${PEAKS:-1}" = "1" ]; then
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/peaks scripts/ubench/peaks.cu && /tmp/peaks > gpurun_out/${TAG}_peaks.json; echo "peaks rc=$?"; cat gpurun_out/${TAG}_peaks.json
fi
if [ "${SWEEP:-1}" = "1" ]; then
timeout 900 python scripts/instance_sweep.py gpurun_out/${TAG}_instance_sweep.jsonl > gpurun_out/${TAG}_sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/${TAG}_sweep.log
fi
