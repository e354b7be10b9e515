mkdir -p gpurun_out
timeout 900 python -m paper_2204_14193_b200.cli bench --precision fp32 --blocks 2048 --gamma 0.2 --bf-counts 0,10,20,50,100,200,500,1000,2000 --report gpurun_out/fig3_fp32.csv > gpurun_out/fig3.log 2>&1; echo fig3=$?
cat gpurun_out/fig3_fp32.csv
timeout 600 python -m paper_2204_14193_b200.cli bench --precision fp64 --blocks 256 --gamma 0.2 --bf-counts 0,100,1000,2000 --report gpurun_out/fig3_fp64.csv >> gpurun_out/fig3.log 2>&1; echo fig3_64=$?
cat gpurun_out/fig3_fp64.csv
