export KB_OPS=gs HHG_GS_KERNEL=wide4
python tools/kbench.py 1 2 7 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gs_front -s 2 -c 1 -o gpurun_out/wide4 python tools/kbench.py 1 2 7 1 > gpurun_out/ncu.log 2>&1
echo rc=$? >> gpurun_out/ncu.log
