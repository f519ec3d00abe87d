# Raster-group sweep of the GEMM (knob gemm_raster) with the K-serpentine on: bench step and per-launch
# DRAM bytes + tensor-pipe activity of the GEMM launches.   usage: bash tools/prof_raster.sh <tag> <cfg> <g...>
TAG=$1; CFG=$2; shift 2
M='dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,regex:sm__pipe_tensor.*cycles_active.*\.(avg|sum)$,sm__cycles_elapsed.avg'
for g in "$@"; do
  python bench.py --config $CFG --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-digest --knob gemm_raster=$g > gpurun_out/${TAG}_bench_${CFG}_g$g.json 2>/dev/null
  timeout 600 ncu --metrics "$M" --clock-control none -k regex:fp8_gemm -s 6 -c 2 --csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline --no-digest --knob gemm_raster=$g \
    > gpurun_out/${TAG}_ncu_${CFG}_g$g.csv 2>/dev/null
done
