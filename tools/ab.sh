# A/B of env settings on the scannetpp bench step: tools/ab.sh "ENV=a" "ENV=b" ... (each run: bench with
# the device legs only; prints ms/step and the per-stage serialised ms)
for cfg in "$@"; do
  env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-naive --no-e2e ${AB_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$cfg" <<'PY'
import json, sys
l = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
st = {k: round(v * 1000, 1) for k, v in l["stage_ms"].items()}
print(f"{sys.argv[1]:40s} ms/step {l['ms_per_step']:.3f} eager {l['eager']['ms_per_step'] if l.get('eager') else None} "
      f"stages_us {st} project_frac {l['stage_hbm']['project']['frac']:.3f}", flush=True)
PY
done
