# round-2 final measurement: GPU suite, smoke, bench line, launch list, ncu of the GS kernel
TAG=${TAG:-r02d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err
python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_(vol_march|gs_items|face_apply|face_gs|face_write|lp_apply|lp_gs_compute|lp_write|zero_slots)" -s 0 -c 300 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
export KB_OPS=gs
python tools/kbench.py 1 2 7 1 > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gs_items" -s 1 -c 1 -o gpurun_out/${TAG}_gs python tools/kbench.py 1 2 7 1 > gpurun_out/ncu2.log 2>&1
KB_ITEMS=1 python tools/gsprof.py 1 2 7 5 > gpurun_out/gsprof_$TAG.log 2>&1
echo done >> gpurun_out/ncu2.log
