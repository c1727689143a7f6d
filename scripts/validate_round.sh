# Round-end validation on one B200: the whole -m gpu suite, smoke(), both bench arms.
# gpurun -- TAG=r02h bash scripts/validate_round.sh   (logs under gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG:-r02h}_smi.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG:-r02h}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG:-r02h}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r02h}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG:-r02h}_smoke.log
timeout 400 python bench.py > gpurun_out/${TAG:-r02h}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG:-r02h}_bench.log
timeout 400 python bench.py --impl reference > gpurun_out/${TAG:-r02h}_bench_ref.log 2>&1
tail -3 gpurun_out/${TAG:-r02h}_pytest_gpu.log; tail -3 gpurun_out/${TAG:-r02h}_smoke.log; tail -2 gpurun_out/${TAG:-r02h}_bench.log | cut -c1-600
