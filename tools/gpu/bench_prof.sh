nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
export KB_OPS=apply,gs
python tools/kbench.py 1 2 7 1 > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gs_items|k_vol_march|k_face_apply|k_face_gs" -s 4 -c 4 -o gpurun_out/r02a python tools/kbench.py 1 2 7 1 > gpurun_out/ncu2.log 2>&1
echo done >> gpurun_out/ncu2.log
