# geometry rates (F=32/64/128) for variant libraries: bash scripts/gpu_geom_variants.sh name ...
mkdir -p gpurun_out
for v in "$@"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2204_14193_b200/_diag/$v.so; fi
  echo "== $v"
  FSE_LIB_PATH=$L timeout 300 python scripts/geom_rates.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(f\"F={d['F']:4d} {d['blocks_per_s']/1e6:8.3f} Mblk/s frac {d['frac_nominal']:.3f}\")
    except Exception: print(l.strip()[:200])"
done
