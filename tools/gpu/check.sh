python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_check.log 2> gpurun_out/bench_check.err
