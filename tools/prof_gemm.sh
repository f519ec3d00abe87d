# usage: bash tools/prof_gemm.sh <tag>   -- full ncu capture of one fp8_gemm launch in the bench step
TAG=${1:-gemm}
B="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp8_gemm -s 4 -c 1 -o gpurun_out/$TAG $B > gpurun_out/$TAG.log 2>&1
tail -3 gpurun_out/$TAG.log
