# full GPU test suite + smoke
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -10
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
