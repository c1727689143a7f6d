for G in 1 2 4 8 16; do
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --groups $G > gpurun_out/grp.json 2>gpurun_out/grp.err || tail -5 gpurun_out/grp.err
  python - "$G" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/grp.json").read().strip().splitlines()[-1])
print("groups", sys.argv[1], "frames/s %.0f"%d["value"], "ms/step %.3f"%d["ms_per_step"], "kk launch ms %.3f"%d["roofline"]["launch_ms"], "launches", d["gpu_launches"])
PY
done
