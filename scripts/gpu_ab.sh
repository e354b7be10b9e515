# robust A/B: interleave variant libraries 3x, 20 timed steps each, report medians
# usage: bash scripts/gpu_ab.sh name1 name2 ...  ("base" = product library)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for d in "$@"; do
    if [ $d = base ]; then L=""; else L="$PWD/paper_2204_14193_b200/_diag/$d.so"; fi
    FSE_LIB_PATH=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --frames 64 > gpurun_out/ab_${d}_$rep.log 2>&1
  done
done
python - "$@" <<'PY'
import json, sys, statistics
for d in sys.argv[1:]:
    v = []
    for rep in (1, 2, 3):
        try:
            v.append(json.loads(open(f"gpurun_out/ab_{d}_{rep}.log").read().strip().splitlines()[-1])["value"] / 1e6)
        except Exception as e:
            pass
    print(f"{d:12s} median {statistics.median(v):.3f} Mblk/s  runs {[round(x, 3) for x in v]}")
PY
