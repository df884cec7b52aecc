python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_(vol_march|gs_items|face_apply|face_gs|face_write|lp_apply|lp_gs_compute|lp_write|zero_slots|front_begin)" -s 0 -c 300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
export KB_OPS=gs
python tools/kbench.py 1 2 7 1 > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gs_items|k_face_gs" -s 4 -c 4 -o gpurun_out/r02_gs python tools/kbench.py 1 2 7 1 > gpurun_out/ncu2.log 2>&1
echo done >> gpurun_out/ncu2.log
