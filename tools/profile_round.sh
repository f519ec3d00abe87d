# Round profile captures (run under gpurun from the repo root):
#   bash tools/profile_round.sh <tag>
# 1. bench lines per config (the numbers; never taken under a profiler)
# 2. launch list of one bench step per config (cold-cache, serialised: compare shares)
# 3. ncu --set full of the GEMM launches of one step (fwd; grouped dX+dW) for c2, c4 and moe,
#    and of the cast kernels of the c2 step
TAG=${1:-r01}
mkdir -p gpurun_out
for CFG in c2 c4 c3 c3w1 c3w1hp moe; do
  timeout 600 python bench.py --config $CFG > gpurun_out/${TAG}_bench_${CFG}.json 2> gpurun_out/${TAG}_bench_${CFG}.err
done
timeout 600 python bench.py --config c4 --fsdp --no-cpu-baseline > gpurun_out/${TAG}_bench_c4_fsdp1.json 2> gpurun_out/${TAG}_bench_c4_fsdp1.err
timeout 600 python bench.py --config c5 --fsdp --no-cpu-baseline > gpurun_out/${TAG}_bench_c5_fsdp1.json 2> gpurun_out/${TAG}_bench_c5_fsdp1.err
for CFG in c2 c4 c3w1 moe; do
  B="python bench.py --config $CFG --steps 2 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"amax|cast|gemm|transpose" -c 80 --csv --log-file gpurun_out/${TAG}_launches_${CFG}.csv $B > gpurun_out/${TAG}_launches_${CFG}.log 2>&1
done
for CFG in c2 c4 moe; do
  B="python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
  # warm-up steps launch 2 GEMMs each: skip them, capture the fwd and the grouped bwd launch of step 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp8_gemm -s 6 -c 2 \
    -o gpurun_out/${TAG}_gemm_${CFG} $B > gpurun_out/${TAG}_gemm_${CFG}.log 2>&1
done
B="python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"amax|cast" -s 6 -c 6 \
  -o gpurun_out/${TAG}_casts_c2 $B > gpurun_out/${TAG}_casts_c2.log 2>&1
B="python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mx_cast" -s 9 -c 3 \
  -o gpurun_out/${TAG}_casts_c4 $B > gpurun_out/${TAG}_casts_c4.log 2>&1
ls -la gpurun_out | tail -40
