mkdir -p gpurun_out
bash scripts/gpu_tests.sh
for v in tma notma tma notma; do
  if [ $v = notma ]; then export FSE_NO_TMA=1; else unset FSE_NO_TMA; fi
  timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --frames 64 > gpurun_out/tma_$v.log 2>&1
  echo "$v $(python -c "import json; d=json.loads(open('gpurun_out/tma_$v.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mblk/s', round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
