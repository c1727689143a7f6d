# K3 A/B on one B200: the persistent bulk-copy-prefetch K3 (default) vs the
# one-shot kernel (KKB_K3_PREFETCH=0); bit identity; the fused-path tests.
mkdir -p gpurun_out; O=gpurun_out/exp_k3pf.txt; : > $O
for v in 1 0 1 0; do
  KKB_K3_PREFETCH=$v timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('pf=$v', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_sequential'])" >> $O
done
KKB_K3_PREFETCH=0 timeout 300 python scripts/k3_pf_check.py /tmp/k0.npy >> $O 2>&1
KKB_K3_PREFETCH=1 timeout 300 python scripts/k3_pf_check.py /tmp/k1.npy >> $O 2>&1
python scripts/k3_pf_check.py --compare /tmp/k0.npy /tmp/k1.npy >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_fused_tc.py tests/test_gpu_engine.py tests/test_gpu_stage1_fused.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2 >> $O
cat $O
