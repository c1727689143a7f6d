for cs in "8 1" "4 2" "4 3" "8 2" "8 3" "16 2" "16 3" "32 2" "2 4"; do
  set -- $cs
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --pipe-chunk $1 --pipe-slots $2 > gpurun_out/pipe.json 2>gpurun_out/pipe.err || tail -3 gpurun_out/pipe.err
  python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/pipe.json").read().strip().splitlines()[-1])
print("chunk", sys.argv[1], "slots", sys.argv[2], "frames/s %.0f"%d["value"], {k: round(v,3) for k,v in d["stage_ms_sequential"].items()})
PY
done
