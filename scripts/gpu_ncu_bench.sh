# ncu evidence for the default bench command and the F=128 kernel
# (each command first exits 0 without ncu; numbers printed under ncu are not bench values)
mkdir -p gpurun_out
K='regex:fast_kernel|class_setup|extrapolate_kernel|pack_trace|spatial_kernel|cfse_kernel'
python bench.py --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
echo launches=$?
CMD="python bench.py --steps 2 --warmup 1 --tiles device --no-e2e --no-cpu --parity-sample 0"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/prof_bench64 $CMD > gpurun_out/ncu_full.log 2>&1
echo full64=$?
python scripts/geom_rates.py 128 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/prof_fast128 python scripts/geom_rates.py 128 > gpurun_out/ncu_full128.log 2>&1
echo full128=$?
