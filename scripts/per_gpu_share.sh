# one rank's share of config 5 at N = 1/2/4/8 GPUs, measured on one B200
# (bench.py --frames 256/128/64/32) -> gpurun_out/per_gpu_share.jsonl
mkdir -p gpurun_out
for f in 256 128 64 32; do
  python bench.py --frames $f --steps 10 --warmup 3 --no-cpu --parity-sample 0 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(json.dumps({'frames_per_gpu': $f, 'gpus_equivalent': 256 // $f, 'device_blocks_per_s': d['value'],
                  'e2e_blocks_per_s': d['e2e']['value'], 'ms_per_step': d['ms_per_step'],
                  'kernel_ms': d['roofline']['kernel_ms'], 'clocks': d['clocks']}))"
done > gpurun_out/per_gpu_share.jsonl
