timeout 600 ncu --set full --clock-control none -c 8 -o gpurun_out/pair python tools/gemm_pair.py > gpurun_out/pair.log 2>&1
tail -2 gpurun_out/pair.log
