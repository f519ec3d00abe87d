mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mx_cast -c 4 -o /tmp/mx python tools/mx_cast_probe.py 16384 28672 > gpurun_out/r02u_mxncu.log 2>&1
python tools/ncu_stalls.py /tmp/mx.ncu-rep > gpurun_out/r02u_mx_stalls.txt 2>&1
ncu -i /tmp/mx.ncu-rep --page source --csv --kernel-name regex:mx_cast_ws -c 1 > gpurun_out/r02u_mx_source.csv 2>&1
ls -la gpurun_out/r02u*
