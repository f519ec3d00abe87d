set -x
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/prof_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp8_gemm -s 4 -c 1 -o gpurun_out/r01_gemm $B > gpurun_out/prof_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cast_tile -s 6 -c 1 -o gpurun_out/r01_cast $B > gpurun_out/prof_cast.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amax_tile -s 6 -c 1 -o gpurun_out/r01_amax $B > gpurun_out/prof_amax.log 2>&1
ls -la gpurun_out
