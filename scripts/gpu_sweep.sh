# chunk sweep of the decomposition (frames per r2c/contract/ifft pass)
for c in 4 8 16 32 400; do
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --chunk $c > gpurun_out/sweep_$c.json 2>&1
  python - "$c" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/sweep_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("chunk", sys.argv[1], "frames/s %.0f"%d["value"], {k: round(v,3) for k,v in d["stage_ms_sequential"].items()})
PY
done
