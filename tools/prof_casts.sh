# ncu --set full of the cast kernels on the c4 (MXFP8) and c3w1 (rowwise) workloads
B4="python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
B3="python bench.py --config c3w1 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mx_cast -s 7 -c 1 -o gpurun_out/r01_mxcast $B4 > gpurun_out/p1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amax_tile -s 6 -c 1 -o gpurun_out/r01_amax_rc $B3 > gpurun_out/p2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cast_tile -s 6 -c 1 -o gpurun_out/r01_cast_rc $B3 > gpurun_out/p3.log 2>&1
ls gpurun_out/*.ncu-rep
