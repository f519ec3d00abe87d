# K-serpentine A/B: bench step time and per-launch DRAM bytes of the GEMMs, c4 and c2, knob gemm_kserp 0 / 1
# usage: bash tools/prof_kserp.sh <tag>
TAG=${1:-kserp}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for cfg in c4 c2; do
  for ks in 0 1; do
    python bench.py --config $cfg --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-digest --knob gemm_kserp=$ks > gpurun_out/${TAG}_bench_${cfg}_k$ks.json 2>/dev/null
    timeout 600 ncu --metrics $M --clock-control none -k regex:fp8_gemm -s 6 -c 2 --csv \
      python bench.py --config $cfg --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline --no-digest --knob gemm_kserp=$ks \
      > gpurun_out/${TAG}_ncu_${cfg}_k$ks.csv 2>/dev/null
  done
done
