# quick A/B of the LS kernels on the GPU box: tools/ab_bench.sh <tag> [ENV=VAL ...]
# runs the default bench workload for 1 timed step, no CPU / e2e legs.
tag=$1; shift
mkdir -p gpurun_out
env "$@" timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_$tag.log 2>&1
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
for l in open(f"gpurun_out/ab_{tag}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        k = {n: round(v["ms"] / v["launches"], 3) for n, v in d["kernels"].items()}
        print(tag, f"{d['value']:.4g}", f"ls_frac={d['ls_roofline']['frac']:.3f}", k)
PY
