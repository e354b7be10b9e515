# parity (GPU) + short bench at 64 frames
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -3
grep -E "^.?config" gpurun_out/pytest_gpu.log | cut -c1-200
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --frames 64 > gpurun_out/bench_q.log 2>&1; echo bench=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mblk/s frac', round(d['roofline']['frac'],3), 'kernel_ms', round(d['roofline']['kernel_ms'],2))"
