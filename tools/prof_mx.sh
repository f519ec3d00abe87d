B4="python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --no-bf16 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mx_cast -s 7 -c 1 -o gpurun_out/r01_mxcast2 $B4 > gpurun_out/p1.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 120 -x -k "mx or linear" 2>&1 | tail -2
