nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err
