# full-step bench sweep over knobs: prints ms/step and per-kernel ms/launch
for kv in "$@"; do
  env $kv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1
  python - "$kv" <<'PY'
import json, sys
d = json.loads(open("/tmp/b.log").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"]), {k: round(v["ms"] / v["launches"], 2) for k, v in d["kernels"].items()})
PY
done
