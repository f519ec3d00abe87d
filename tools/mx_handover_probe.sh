export PROBE_SHAPES=16384x28672x8192,16384x14336x4096 PROBE_KINDS=mx PROBE_MODES=0,8,1
python tools/gemm_bound_probe.py > gpurun_out/r02q_probe_mx.txt 2>&1
