# ncu evidence for the fused kernel (run only after the same commands exited 0 plainly)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --frames 32"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/prof_fast64 $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
tail -3 gpurun_out/ncu_full.log
