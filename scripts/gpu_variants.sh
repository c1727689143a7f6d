# bench each tuning variant of libkkb (no e2e / cpu legs)
for lib in paper_2603_22496_b200/libkkb.so paper_2603_22496_b200/variants/libkkb_*.so; do
  KKB_LIB=$PWD/$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/var.json 2>gpurun_out/var.err || tail -3 gpurun_out/var.err
  python - "$lib" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/var.json").read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], "frames/s %.0f"%d["value"], {k: round(v,3) for k,v in d["stage_ms_sequential"].items()})
PY
done
