# bench variant libraries: bash scripts/gpu_variants.sh name1 name2 ... (paper_2204_14193_b200/_diag/<name>.so; "base" = product)
mkdir -p gpurun_out
for d in "$@"; do
  if [ $d = base ]; then L=""; else L="$PWD/paper_2204_14193_b200/_diag/$d.so"; fi
  FSE_LIB_PATH=$L timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --frames 64 > gpurun_out/var_$d.log 2>&1
  echo "$d $(python -c "import json,sys; d=json.loads(open('gpurun_out/var_$d.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mblk/s', round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
