# Round profile captures (run under gpurun from the repo root):
#   bash tools/profile_round.sh <tag>
# 1. launch list of one bench step per config (cold-cache, serialised: compare shares)
# 2. ncu --set full of the top kernel (GEMM) and the cast kernels of the c2 step
TAG=${1:-r01}
mkdir -p gpurun_out
for CFG in c2 c4 c3w1; do
  B="python bench.py --config $CFG --steps 2 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"amax|cast|gemm|transpose" -c 60 --csv --log-file gpurun_out/${TAG}_launches_${CFG}.csv $B > gpurun_out/${TAG}_launches_${CFG}.log 2>&1
done
B="python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp8_gemm -s 3 -c 3 \
  -o gpurun_out/${TAG}_gemm_c2 $B > gpurun_out/${TAG}_gemm_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"amax|cast" -s 6 -c 6 \
  -o gpurun_out/${TAG}_casts_c2 $B > gpurun_out/${TAG}_casts_c2.log 2>&1
ls -la gpurun_out | tail -20
