mkdir -p gpurun_out
for s in 0 8000 20000 32000 50000; do
  FSE_STAGGER_NS=$s timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --frames 64 > gpurun_out/stg_$s.log 2>&1
  echo "stagger=$s $(python -c "import json,sys; d=json.loads(open('gpurun_out/stg_$s.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mblk/s', round(d['roofline']['frac'],3))")"
done
