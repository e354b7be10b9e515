# full bench + ncu --set full capture of the fused kernel (tag = $1)
mkdir -p gpurun_out
TAG=${1:-cur}
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3),'Mblk/s frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value']/1e6,3), 'cpu', d.get('cpu_baseline',{}).get('value'))"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --frames 32"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$?
