# A/B of runtime environment settings on the product library:
# bash scripts/gpu_ab_env.sh "NAME=VAR=VALUE" ...   ("base" = no extra env)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for spec in "$@"; do
    n=${spec%%=*}; e=${spec#*=}
    if [ "$spec" = base ]; then n=base; e=""; fi
    env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --frames 64 > gpurun_out/abe_${n}_$rep.log 2>&1
  done
done
python - "$@" <<'PY'
import json, sys, statistics
for spec in sys.argv[1:]:
    n = "base" if spec == "base" else spec.split("=")[0]
    v = []
    for rep in (1, 2, 3):
        try:
            v.append(json.loads(open(f"gpurun_out/abe_{n}_{rep}.log").read().strip().splitlines()[-1])["value"] / 1e6)
        except Exception:
            pass
    print(f"{n:12s} median {statistics.median(v):.3f} Mblk/s  runs {[round(x, 3) for x in v]}")
PY
