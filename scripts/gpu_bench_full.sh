mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log
