# Round profile artefacts (run under gpurun; summarise here with tools/ncu_summary.py / ncu_traffic.py):
#   launch lists of the headline (c4), c2 and c3 steps; ncu --set full of the c4 / c2 GEMM launches, the c4 MX
#   casts, the c2 amax / casts and the c3 row / column amax + multi-tensor casts.
# usage: bash tools/round_profile.sh <tag>
T=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline --no-digest"
for c in c4 c2 c3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:fp8t:: --csv --log-file gpurun_out/${T}_launches_$c.csv \
    $B --config $c > gpurun_out/${T}_launches_$c.log 2>&1
done
B1="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline --no-digest"
timeout 1200 ncu --set full --metrics sm__pipe_tensor_cycles_active.avg,sm__cycles_elapsed.avg --clock-control none --import-source on -k regex:fp8_gemm -s 6 -c 2 -o gpurun_out/${T}_gemm_c4 $B1 --config c4 > gpurun_out/${T}_gemm_c4.log 2>&1
timeout 1200 ncu --set full --metrics sm__pipe_tensor_cycles_active.avg,sm__cycles_elapsed.avg --clock-control none --import-source on -k regex:fp8_gemm -s 6 -c 2 -o gpurun_out/${T}_gemm_c2 $B1 --config c2 > gpurun_out/${T}_gemm_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mx_cast -s 9 -c 3 -o gpurun_out/${T}_casts_c4 $B1 --config c4 > gpurun_out/${T}_casts_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"amax|cast" -s 12 -c 4 -o gpurun_out/${T}_casts_c2 $B1 --config c2 > gpurun_out/${T}_casts_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"amax_rc|cast_tile" -s 32 -c 4 -o gpurun_out/${T}_casts_c3 $B1 --config c3 > gpurun_out/${T}_casts_c3.log 2>&1
ls -la gpurun_out/${T}_*
