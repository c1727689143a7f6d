# compute-sanitizer over the product kernels on one B200 (memcheck, racecheck,
# synccheck, initcheck) running smoke(): config-1 stage 1 + FMA gather + taps +
# DAS, then the 48-frame config-4 bench path (fused stage 1 -> tcgen05 gather).
#   gpurun -- bash scripts/sanitize.sh      (summaries under gpurun_out/)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke:" gpurun_out/sanitize_$tool.log | tee -a gpurun_out/sanitize_summary.txt
done
