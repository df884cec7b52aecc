timeout 1700 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
