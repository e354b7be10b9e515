# bench line + ncu launch list + ncu full capture of the fused kernel (current build)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_final.log | cut -c1-400
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --frames 32"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launches3.log 2>&1; echo launches=$?
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/prof_final $CMD > gpurun_out/ncu_full4.log 2>&1; echo full=$?
